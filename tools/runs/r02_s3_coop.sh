mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/co_smoke.log 2>&1; tail -3 gpurun_out/co_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/co_bench.json 2> gpurun_out/co_bench.err; python tools/bsum.py gpurun_out/co_bench.json; tail -2 gpurun_out/co_bench.err
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/co_tests.log 2>&1; tail -3 gpurun_out/co_tests.log
echo done
