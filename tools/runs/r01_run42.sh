# adaptive blind-backoff cap (GC_BACKOFF_LO, GC_BACKOFF_LO_CAP), all six non-deterministic schemes
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,to,mvcc,silo,tictoc
probe() {
  timeout 300 python tools/probe.py --reps 3 --schemes $S --thetas 0.6,0.8 --seeds 3 --lanes 16 --grid 148 --bs 16 > gpurun_out/bpace_$1_ycsb.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs 1 --grid 148 --reps 2 --schemes $S > gpurun_out/bpace_$1_tpcc1.log 2>&1
  timeout 300 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs 8 --grid 148 --reps 2 --schemes $S > gpurun_out/bpace_$1_tpcc64.log 2>&1
}
probe base
for V in "b32c7:-DGC_BACKOFF_LO=32" "b32c8:-DGC_BACKOFF_LO=32 -DGC_BACKOFF_LO_CAP=8u" "b128c7:-DGC_BACKOFF_LO=128"; do
  name=${V%%:*}; flags=${V#*:}
  GCCTB_NVCC_EXTRA="$flags" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
  probe $name
done
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
