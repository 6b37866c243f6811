mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
GCCTB_LIB=$PWD/variants/fifo_trace.so timeout 600 python tools/trace_tail.py --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.6 --bucket_ns 5000 > gpurun_out/s3_trace_fifo2.jsonl 2>&1
cut -c1-250 gpurun_out/s3_trace_fifo2.jsonl
export GCCTB_LIB=$PWD/variants/fifo.so
( timeout 900 python tools/probe.py --reps 3 --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0,0.6,0.8,0.9,0.99 --lanes 16 --bs 16 --grid 148 --watchdog 60 2>&1 | cut -c1-330
  timeout 900 python tools/probe.py --reps 2 --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.6,0.9 --lanes 1 --wd 5 --bs 8 --watchdog 60 2>&1 | cut -c1-330 ) > gpurun_out/s3_probe_fifo2.log
unset GCCTB_LIB
cat gpurun_out/s3_probe_fifo2.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l[:l.index(', \"ms_total_min')]+'}')
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], d['lanes'], round(d['txn_s']/1e6,2), round(d['abort_rate'],2), round(d['ms_total_median'],3))
"
echo done
