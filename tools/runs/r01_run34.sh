# one transaction per warp (32-lane tiles) vs two per warp (16): does a sleeping warp-mate delay the other tile?
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 3 --thetas 0.6,0.8 --lanes 16 --grid 148 --bs 16 --seeds 3 > gpurun_out/lanes16.log 2>&1
timeout 600 python tools/probe.py --reps 3 --thetas 0.6,0.8 --lanes 32 --grid 148 --bs 32 --seeds 3 > gpurun_out/lanes32.log 2>&1
timeout 600 python tools/probe.py --reps 3 --thetas 0.6,0.8 --lanes 32 --grid 0 --bs 32 --seeds 3 > gpurun_out/lanes32full.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "c1_parity or brute" > gpurun_out/t34.log 2>&1; tail -1 gpurun_out/t34.log
echo done
