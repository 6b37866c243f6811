mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in fifo_h64 fifo_h256 fifo_h1024; do
  export GCCTB_LIB=$PWD/variants/$v.so
  echo "# $v"
  timeout 900 python tools/probe.py --reps 3 --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0,0.6,0.8,0.9,0.99 --lanes 16 --bs 16 --grid 148 --watchdog 60 2>&1 | cut -c1-330
  timeout 900 python tools/probe.py --reps 2 --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.6,0.9 --lanes 1 --wd 5 --bs 8 --watchdog 60 2>&1 | cut -c1-330
done > gpurun_out/s3_probe_fifo5.log
unset GCCTB_LIB
cat gpurun_out/s3_probe_fifo5.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l[:l.index(', \"ms_total_min')]+'}')
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], d['lanes'], round(d['txn_s']/1e6,2), round(d['abort_rate'],2), round(d['ms_total_median'],3))
"
echo done
