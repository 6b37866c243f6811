# TPC-C configs[4] shape on one GPU (512 warehouses, 64K batch, 45:43 mix): launch sweep
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for g in "8 0" "16 0" "32 0" "8 148" "16 148" "32 148"; do set -- $g
  timeout 900 python tools/probe_tpcc.py --W 512 --batch 65536 --mix 5114 --bs $1 --grid $2 --reps 2
done > gpurun_out/tpcc_c5.log 2>&1
echo done
