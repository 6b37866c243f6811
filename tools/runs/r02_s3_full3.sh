mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/f3_smoke.log 2>&1; tail -1 gpurun_out/f3_smoke.log
B="python bench.py --steps 20 --warmup 5 --no-tpcc --no-cpu-baseline --no-index-binary"
for r in 1 2; do
  $B > gpurun_out/f3_b_main$r.json 2>/dev/null; python tools/bsum.py gpurun_out/f3_b_main$r.json | head -1
  GCCTB_LIB=$PWD/variants/zmemset.so $B > gpurun_out/f3_b_zm$r.json 2>/dev/null; python tools/bsum.py gpurun_out/f3_b_zm$r.json | head -1
done
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/f3_tests.log 2>&1; tail -3 gpurun_out/f3_tests.log
echo done
