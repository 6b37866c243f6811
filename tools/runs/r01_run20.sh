# GPUTx / GaccO: fewer resident tiles (grid 148 x bs warps) -- polling pressure vs parallelism
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for bs in 4 8 16 32; do
  timeout 300 python tools/probe.py --reps 3 --schemes gputx,gacco --thetas 0.6 --lanes 16 --grid 148 --bs $bs
done > gpurun_out/det_grid.log 2>&1
echo done
