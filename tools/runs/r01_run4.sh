mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/probe_tpcc.py --W 1 --lanes 32 --watchdog 20 --reps 2 > gpurun_out/tpcc_w1_v4.log 2>&1
timeout 900 python tools/probe.py --thetas 0,0.6,0.9,0.99 --lanes 16 --reps 3 > gpurun_out/probe_v4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -k "c1 or c2 or c3 or c4 or pipeline or prepare or prepared or brute or partition or smoke" > gpurun_out/gpu_tests4.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_tests4.log
timeout 600 python bench.py > gpurun_out/bench4.log 2>&1
timeout 600 python bench.py --no-pipeline > gpurun_out/bench4_nopipe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/prof_dense python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_dense.log 2>&1
echo done
