export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_ycsb.py -m gpu -q --timeout 900 -k "bench_launch and gputx" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin7_bench.json 2>gpurun_out/fin7_bench.err; python tools/bsum.py gpurun_out/fin7_bench.json 2>/dev/null
