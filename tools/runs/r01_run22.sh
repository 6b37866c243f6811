# per-scheme launch tuning at the bench workload (theta 0.6): warps per SM (1 block/SM)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for bs in 6 8 12 16 24 32; do
  timeout 300 python tools/probe.py --reps 3 --thetas 0.6 --lanes 16 --grid 148 --bs $bs --seeds 3,5
done > gpurun_out/tune_bs.log 2>&1
echo done
