mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin4_smoke.log 2>&1; tail -1 gpurun_out/fin4_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin4_bench.json 2> gpurun_out/fin4_bench.err; python tools/bsum.py gpurun_out/fin4_bench.json 2>/dev/null | head -1
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin4_tests.log 2>&1; tail -3 gpurun_out/fin4_tests.log
echo done
