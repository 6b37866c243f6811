mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in 14 12 10; do
  GCCTB_TO_BACKOFF_CAP=$c timeout 600 python tools/probe.py --reps 5 --seeds 1003,1005,1006 --thetas 0.6 --lanes 16 --schemes to,mvcc > gpurun_out/tocap_${c}_mc.log 2>&1
  GCCTB_TO_BACKOFF_CAP=$c timeout 900 python tools/probe.py --reps 2 --watchdog 60 --thetas 0.8,0.9,0.95,0.99 --lanes 16 --schemes to,mvcc > gpurun_out/tocap_${c}_hc.log 2>&1
  GCCTB_TO_BACKOFF_CAP=$c timeout 600 python tools/probe.py --reps 2 --watchdog 60 --thetas 0.9,0.99 --lanes 1 --schemes to > gpurun_out/tocap_${c}_thread.log 2>&1
done
echo done
