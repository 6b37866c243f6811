mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 3 --thetas 0,0.6 --lanes 16 > gpurun_out/probe_v17.log 2>&1
timeout 600 python bench.py > gpurun_out/bench13.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests13.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests13.log
echo done
