export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_ycsb.py -m gpu -q --timeout 900 -k "bench_launch" 2>&1 | tail -3
