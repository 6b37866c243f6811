mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 2; do
timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "2pc" 2>&1 | tail -4
GCCTB_LIB=$PWD/variants/nocoop.so timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q --timeout 600 -k "2pc" 2>&1 | tail -4
done
