mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
fails=0
for i in $(seq 1 40); do
  timeout 600 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 300 -k "test_loopback_2pc" -x > gpurun_out/fl4_$i.log 2>&1 || { fails=$((fails+1)); cp gpurun_out/fl4_$i.log gpurun_out/fl4_fail_$i.log; }
  rm -f gpurun_out/fl4_$i.log
done
echo "fails=$fails of 40 runs (each the 12 loopback 2PC tests)"
ls gpurun_out/fl4_fail_* 2>/dev/null | head
