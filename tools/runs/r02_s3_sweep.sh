mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python tools/sweep.py theta --reps 2 --budget-ms 400 --out gpurun_out/r02_sweep_theta_final.jsonl > gpurun_out/sw_theta.log 2>&1; tail -2 gpurun_out/sw_theta.log
timeout 1800 python tools/sweep.py stages --out gpurun_out/r02_sweep_stages_final.jsonl > gpurun_out/sw_stages.log 2>&1; tail -2 gpurun_out/sw_stages.log
wc -l gpurun_out/r02_sweep_*_final.jsonl
