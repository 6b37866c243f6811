# GPUTx rank pass: max_rank from the sort (no per-txn atomicMax); poll cap sweep
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "gputx" > gpurun_out/t27.log 2>&1; tail -1 gpurun_out/t27.log
for poll in 32 128 512; do echo "# poll=$poll"; GCCTB_RANK_POLL_NS=$poll timeout 300 python tools/probe.py --reps 3 --schemes gputx --thetas 0.6,0.8 --lanes 16 --grid 148 --bs 8; done > gpurun_out/rank_sweep3.log 2>&1
echo done
