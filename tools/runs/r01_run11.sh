mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 3 --watchdog 60 --schemes to --thetas 0.6,0.8,0.9,0.95,0.99 --lanes 16 > gpurun_out/to_v11.log 2>&1
echo done
