mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
P="timeout 300 python tools/probe.py --reps 1 --watchdog 120 --schemes tpl_wd"
$P --thetas 0.8,0.9 --lanes 16 > gpurun_out/wd_tile.log 2>&1
$P --thetas 0.9 --lanes 16 --flags 0x200 > gpurun_out/wd_tile_flat.log 2>&1
$P --thetas 0.9 --lanes 1 > gpurun_out/wd_thread.log 2>&1
$P --thetas 0.9 --lanes 4 > gpurun_out/wd_tile4.log 2>&1
timeout 300 python tools/probe.py --reps 1 --watchdog 120 --schemes tpl_wd --thetas 0.9 --lanes 16 --flags 0x1 > gpurun_out/wd_tile_immediate.log 2>&1
echo done
