# adaptive post-wait jitter cap (GC_JITTER_LO, GC_JITTER_LO_SHIFT)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,silo,tictoc
probe() {
  timeout 300 python tools/probe.py --reps 3 --schemes $S --thetas 0.6,0.8 --seeds 3 --lanes 16 --grid 148 --bs 16 > gpurun_out/apace_$1_ycsb.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs 1 --grid 148 --reps 2 --schemes $S > gpurun_out/apace_$1_tpcc1.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs 8 --grid 148 --reps 2 --schemes $S > gpurun_out/apace_$1_tpcc64.log 2>&1
}
probe base
for V in "a32:-DGC_JITTER_LO=32" "a128:-DGC_JITTER_LO=128" "a512:-DGC_JITTER_LO=512" "a128s7:-DGC_JITTER_LO=128 -DGC_JITTER_LO_SHIFT=7"; do
  name=${V%%:*}; flags=${V#*:}
  GCCTB_NVCC_EXTRA="$flags" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
  probe $name
done
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
