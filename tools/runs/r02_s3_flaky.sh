mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
echo "# new"
timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "test_loopback_2pc and (to or mvcc or silo or tictoc)" --count 1 2>/dev/null | tail -2
for i in 1 2 3 4 5 6; do timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "test_loopback_2pc and (to or mvcc or silo or tictoc)" 2>&1 | tail -1; done
echo "# old"
cd variants/oldtree
for i in 1 2 3 4 5 6; do timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "test_loopback_2pc and (to or mvcc or silo or tictoc)" 2>&1 | tail -1; done
