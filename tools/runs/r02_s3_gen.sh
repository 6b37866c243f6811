mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/gen_smoke.log 2>&1; tail -2 gpurun_out/gen_smoke.log
timeout 900 python -m pytest tests/test_gpu_ycsb.py -m gpu -q --timeout 600 -k "gen or generator or c1_parity or c2" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/gen_bench.json 2> gpurun_out/gen_bench.err; python tools/bsum.py gpurun_out/gen_bench.json; tail -2 gpurun_out/gen_bench.err
