mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/probe.py --thetas 0,0.6,0.9,0.99 --lanes 16 --reps 3 > gpurun_out/probe_v5.log 2>&1
timeout 900 python tools/probe_tpcc.py --W 1 --lanes 32 --watchdog 20 --reps 2 > gpurun_out/tpcc_w1_v5.log 2>&1
timeout 600 python bench.py > gpurun_out/bench5.log 2>&1
timeout 600 python bench.py --no-pipeline > gpurun_out/bench5_nopipe.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests5.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/gpu_tests5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/prof_v5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_v5.log 2>&1
echo done
