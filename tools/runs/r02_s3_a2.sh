mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/a2_smoke.log 2>&1; tail -3 gpurun_out/a2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/a2_bench.json 2> gpurun_out/a2_bench.err; python tools/bsum.py gpurun_out/a2_bench.json; tail -2 gpurun_out/a2_bench.err
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -k "mvcc or partition or multiproc or pipeline or c1_parity or error or generator" > gpurun_out/a2_tests.log 2>&1; tail -3 gpurun_out/a2_tests.log
echo done
