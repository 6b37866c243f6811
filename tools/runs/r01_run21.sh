# GPUTx: K-set sleep ~ distance x 1.5 us; rank-pass poll cap / grid divisor sweep
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for poll in 128 512 2048; do for div in 1 4; do
  echo "# poll=$poll div=$div"
  GCCTB_RANK_POLL_NS=$poll GCCTB_RANK_GRID_DIV=$div timeout 300 python tools/probe.py --reps 3 --schemes gputx --thetas 0.6,0.8 --lanes 16
done; done > gpurun_out/rank_sweep.log 2>&1
timeout 300 python tools/probe.py --reps 3 --schemes gputx --thetas 0.6 --lanes 16 --grid 148 --bs 8 >> gpurun_out/rank_sweep.log 2>&1
echo done
