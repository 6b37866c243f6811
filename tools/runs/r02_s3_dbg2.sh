export PYTHONUNBUFFERED=1
for s in to silo tictoc mvcc; do timeout 900 python tools/dbg_2pc.py $s 50 2>&1 | tail -4; done
