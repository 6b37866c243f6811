mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in nocoop nofifo; do
echo "# $v"
export GCCTB_LIB=$PWD/variants/$v.so
for i in 1 2 3 4 5 6 7 8; do timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "test_loopback_2pc and (to or mvcc or silo or tictoc)" 2>&1 | grep -E "passed|FAILED"; done
done
