# occupancy vs contention for the lock/OCC/TO schemes in tile mode: theta 0 vs 0.6 at 8/16/32 warps per SM (1 block/SM) and the full grid
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,to,mvcc,silo,tictoc
for bs in 8 16 32; do
  timeout 300 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 16 --grid 148 --bs $bs > gpurun_out/occ_g148_bs$bs.log 2>&1
done
timeout 300 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 16 --grid 0 --bs 32 > gpurun_out/occ_full.log 2>&1
echo done
