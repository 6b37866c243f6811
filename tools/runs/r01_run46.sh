# re-tune warps per SM (one block per SM) after the adaptive pacing change, theta=0.6 (bench) and 0.8
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for bs in 12 16 20 24 32; do
  timeout 300 python tools/probe.py --reps 5 --schemes tpl_nw,tpl_wd,to,mvcc,silo,tictoc --thetas 0.6 --seeds 3,5 --lanes 16 --grid 148 --bs $bs > gpurun_out/tune46_bs$bs.log 2>&1
done
echo done
