mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 5 --seeds 1003,1005,1006 --thetas 0.6 --lanes 16 --schemes to,mvcc > gpurun_out/toad_mc.log 2>&1
timeout 900 python tools/probe.py --reps 2 --watchdog 60 --thetas 0.8,0.9,0.95,0.99 --lanes 16 --schemes to,mvcc > gpurun_out/toad_hc.log 2>&1
timeout 600 python tools/probe.py --reps 2 --watchdog 60 --thetas 0.9,0.99 --lanes 1 --schemes to > gpurun_out/toad_thread.log 2>&1
timeout 300 python tools/probe_tpcc.py --W 1 --lanes 32 --watchdog 30 --reps 2 --schemes to,mvcc > gpurun_out/toad_tpcc.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench16.log 2>&1
echo done
