mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/last_smoke.log 2>&1; tail -1 gpurun_out/last_smoke.log
timeout 1800 python -m pytest tests/test_gpu_ycsb.py tests/test_gpu_pipeline.py tests/test_gpu_partition.py -m gpu -q --timeout 900 -x 2>&1 | tail -1
for v in main grelax; do
  if [ $v = main ]; then unset GCCTB_LIB; else export GCCTB_LIB=$PWD/variants/$v.so; fi
  echo "# $v"; timeout 600 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6,0.8 --lanes 32 --bs 8 --grid 148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], 'exec', round(d['ms_exec_median'],3))
"; done
unset GCCTB_LIB
timeout 900 python bench.py --steps 20 --warmup 5 --no-tpcc --no-cpu-baseline > gpurun_out/last_bench.json 2>/dev/null; python tools/bsum.py gpurun_out/last_bench.json 2>/dev/null | head -1
