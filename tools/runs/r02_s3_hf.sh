mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in trace hf8 hf100000; do
  export GCCTB_LIB=$PWD/variants/$v.so
  echo "# $v"
  for r in 1 2; do timeout 600 python tools/trace_tail.py --schemes tpl_nw,silo,tictoc --thetas 0.6 --bucket_ns 5000 2>&1 | cut -c1-200; done
  timeout 600 python tools/trace_tail.py --schemes tpl_nw,silo,tictoc --thetas 0.8 --bucket_ns 20000 2>&1 | cut -c1-200
  timeout 600 python tools/trace_tail.py --schemes tpl_nw,silo,tictoc --thetas 0.99 --bucket_ns 200000 2>&1 | cut -c1-200
  timeout 600 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --schemes tpl_nw,silo,tictoc --lanes 32 --reps 2 --watchdog 60 2>&1 | cut -c1-250
done > gpurun_out/s3_hf.log
cat gpurun_out/s3_hf.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l[:l.index(', \"commits_hist')]+'}'); print(d['scheme'], d['theta'], round(d['exec_ms'],3), d['t99_us'], d['t100_us']); continue
    except Exception: pass
    print(l[:250].strip())
"
