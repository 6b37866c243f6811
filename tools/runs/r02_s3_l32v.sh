mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/l32_smoke.log 2>&1; tail -1 gpurun_out/l32_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/l32_bench.json 2> gpurun_out/l32_bench.err; python tools/bsum.py gpurun_out/l32_bench.json
timeout 2400 python -m pytest tests/test_gpu_ycsb.py -m gpu -q --timeout 900 -k "bench_launch or c1_parity" > gpurun_out/l32_tests.log 2>&1; tail -2 gpurun_out/l32_tests.log
timeout 1500 python tools/probe_hc.py --thetas 0.6,0.8,0.9,0.95,0.99 --tag l32 > gpurun_out/l32_hc.jsonl 2>&1; tail -1 gpurun_out/l32_hc.jsonl
