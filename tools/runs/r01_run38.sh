# CC_FLAG_WARM (0x2000): lines in L2 before the first CC step -- parity + tuned-launch probes
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ycsb.py -m gpu -q -k "warm" > gpurun_out/t38_warm.log 2>&1; tail -1 gpurun_out/t38_warm.log
for s in tpl_nw tpl_wd to mvcc silo tictoc; do
  bs=16; [ $s = tictoc ] && bs=12
  for f in 0 0x2000; do
    timeout 300 python tools/probe.py --reps 5 --schemes $s --thetas 0,0.6,0.8 --seeds 3 --lanes 16 --grid 148 --bs $bs --flags $f >> gpurun_out/warm_$f.log 2>&1
  done
done
echo done
