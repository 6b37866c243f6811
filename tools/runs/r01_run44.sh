# GaccO: two acquire polls in flight for the next-in-line waiter (GC_GACCO_POLL2 = gap ns)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
probe() {
  timeout 300 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6,0.8 --seeds 3,5 --lanes 16 --grid 148 --bs 24 > gpurun_out/poll2_$1.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs 16 --grid 148 --reps 2 --schemes gacco >> gpurun_out/poll2_$1.log 2>&1
}
probe base
for V in "p150:-DGC_GACCO_POLL2=150" "p300:-DGC_GACCO_POLL2=300" "p500:-DGC_GACCO_POLL2=500"; do
  name=${V%%:*}; flags=${V#*:}
  GCCTB_NVCC_EXTRA="$flags" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
  probe $name
done
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
