# GaccO / GPUTx far-waiter sleep cap (GC_GACCO_MAX_SLEEP_NS, GC_KSET_MAX_SLEEP_NS) and GaccO hop estimate
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
probe() {
  timeout 300 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6,0.8 --seeds 3,5 --lanes 16 --grid 148 --bs 24 > gpurun_out/sl_$1_gacco.log 2>&1
  timeout 300 python tools/probe.py --reps 3 --schemes gputx --thetas 0.6,0.8 --seeds 3,5 --lanes 16 --grid 148 --bs 8 > gpurun_out/sl_$1_gputx.log 2>&1
}
probe base
for V in "s2000:-DGC_GACCO_MAX_SLEEP_NS=2000u -DGC_KSET_MAX_SLEEP_NS=2000u" "s8000:-DGC_GACCO_MAX_SLEEP_NS=8000u -DGC_KSET_MAX_SLEEP_NS=8000u" "s2000h300:-DGC_GACCO_MAX_SLEEP_NS=2000u -DGC_KSET_MAX_SLEEP_NS=2000u -DGC_GACCO_HOP_NS=300"; do
  name=${V%%:*}; flags=${V#*:}
  GCCTB_NVCC_EXTRA="$flags" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
  probe $name
done
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
