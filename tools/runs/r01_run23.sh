mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 700 python -m pytest tests -m gpu -x -q -k "gputx or roofline or pipeline" > gpurun_out/t23.log 2>&1; tail -2 gpurun_out/t23.log
for div in 1 2; do echo "# extra div=$div"; GCCTB_RANK_GRID_DIV=$div timeout 300 python tools/probe.py --reps 3 --schemes gputx --thetas 0.6,0.8 --lanes 16 --grid 148 --bs 8; done > gpurun_out/rank_sweep2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_tuned.json 2> gpurun_out/bench_tuned.err
echo done
