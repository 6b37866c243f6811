mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench14_$i.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench14_10.log 2>&1
timeout 600 python tools/probe.py --reps 5 --seeds 1003,1004,1005,1006,1007 --thetas 0.6 --lanes 16 > gpurun_out/probe_seeds14.log 2>&1
echo done
