import sys; sys.path.insert(0,'.')
import numpy as np, torch, inputs
from paper_2406_10158_b200.api import DB
from paper_2406_10158_b200 import gcctb as G
db=DB(0); db.load_ycsb(1<<20, 1)
T=inputs.zipf_thresholds(1<<20, 0.6); A=inputs.scramble_mult(1<<20)
b=db.gen_ycsb(65536,16,0.1,1,T,A)
for lanes,bs,grid,wd in [(16,16,148,0),(16,32,0,0),(16,8,148,0),(1,32,0,0),(1,32,0,5),(4,32,0,0),(32,16,148,0)]:
    for s in ["tpl_nw","mvcc","gacco","gputx"]:
        try:
            r=db.submit(b,s,wd=wd,bs=bs,grid=grid,lanes=lanes); st=db.sync(); print(lanes,bs,grid,wd,s,"ok",st.commits)
        except Exception as e: print(lanes,bs,grid,wd,s,"ERR",e)
