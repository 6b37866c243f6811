mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/probe_tpcc.py --W 1 --lanes 32 --watchdog 20 --reps 2 > gpurun_out/tpcc_w1_v3.log 2>&1
timeout 900 python tools/probe.py --thetas 0.6,0.9,0.99 --lanes 16 --reps 3 > gpurun_out/probe_v3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --no-pipeline > gpurun_out/bench_nopipe.log 2>&1
echo done
