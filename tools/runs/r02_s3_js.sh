mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in trace js4 js6; do
  export GCCTB_LIB=$PWD/variants/$v.so
  echo "# $v"
  for r in 1 2; do timeout 600 python tools/trace_tail.py --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.6 --bucket_ns 5000 2>&1 | cut -c1-200; done
  timeout 600 python tools/trace_tail.py --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.8 --bucket_ns 20000 2>&1 | cut -c1-200
done > gpurun_out/s3_js.log
cat gpurun_out/s3_js.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l[:l.index(', \"commits_hist')]+'}')
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], round(d['exec_ms'],3), d['t99_us'], d['t100_us'])
"
