# TPC-C configs[2] (1 warehouse, 16K, 50/50) and configs[3] (64 warehouses) with the current code; launch sweep
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for g in "8 0" "8 148" "4 148" "2 148" "1 148"; do set -- $g
  timeout 600 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --bs $1 --grid $2 --reps 2
done > gpurun_out/tpcc_c3.log 2>&1
for g in "8 0" "8 148" "4 148"; do set -- $g
  timeout 600 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs $1 --grid $2 --reps 2
done > gpurun_out/tpcc_c4.log 2>&1
echo done
