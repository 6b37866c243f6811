mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 3 --watchdog 60 --schemes tpl_wd,tpl_nw --thetas 0.6,0.8,0.9,0.95,0.99 --lanes 16 > gpurun_out/wd_v12.log 2>&1
timeout 300 python tools/probe_tpcc.py --W 1 --lanes 32 --watchdog 30 --reps 2 --schemes tpl_wd,to > gpurun_out/wd_tpcc_v12.log 2>&1
echo done
