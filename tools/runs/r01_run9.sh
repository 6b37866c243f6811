mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_partition.py -m gpu -q -rf --timeout 600 > gpurun_out/t9_part.log 2>&1; echo "part rc=$?"; tail -4 gpurun_out/t9_part.log
timeout 900 python bench.py --workload tpcc --loopback 4 --two-pc --schemes tpl_nw,tpl_wd --no-cpu-baseline > gpurun_out/bench9_lb4_2pc.log 2>&1
timeout 900 python bench.py --workload tpcc --loopback 4 --schemes tpl_nw,tpl_wd --no-cpu-baseline > gpurun_out/bench9_lb4_det.log 2>&1
echo done
