# GaccO distance-proportional waits
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "gacco" > gpurun_out/t31.log 2>&1; tail -1 gpurun_out/t31.log
for g in "32 0" "24 148" "8 148"; do set -- $g
 timeout 300 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6,0.8,0.9 --lanes 16 --bs $1 --grid $2
done > gpurun_out/gacco31.log 2>&1
for g in "8 0" "8 148" "4 148" "1 148"; do set -- $g
  timeout 600 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs $1 --grid $2 --reps 2 --schemes gacco
  timeout 600 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs $1 --grid $2 --reps 2 --schemes gacco
done > gpurun_out/gacco31_tpcc.log 2>&1
echo done
