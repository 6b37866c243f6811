# retry pacing caps for the lock / OCC schemes: post-wait jitter (GC_JITTER_MAX_SHIFT) and blind backoff (GC_BACKOFF_CAP)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,silo,tictoc
probe() {
  timeout 300 python tools/probe.py --reps 3 --schemes $S --thetas 0.6,0.8 --seeds 3 --lanes 16 --grid 148 --bs 16 > gpurun_out/pace_$1_ycsb.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs 1 --grid 148 --reps 2 --schemes $S > gpurun_out/pace_$1_tpcc1.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs 8 --grid 148 --reps 2 --schemes $S > gpurun_out/pace_$1_tpcc64.log 2>&1
}
probe base
for V in "j6:-DGC_JITTER_MAX_SHIFT=6" "j8:-DGC_JITTER_MAX_SHIFT=8" "b7:-DGC_BACKOFF_CAP=7u" "j8b8:-DGC_JITTER_MAX_SHIFT=8 -DGC_BACKOFF_CAP=8u"; do
  name=${V%%:*}; flags=${V#*:}
  GCCTB_NVCC_EXTRA="$flags" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
  probe $name
done
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
