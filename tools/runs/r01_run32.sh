mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t32.log 2>&1; tail -1 gpurun_out/t32.log
timeout 600 python bench.py > gpurun_out/bench32.json 2> gpurun_out/bench32.err
timeout 900 python bench.py --workload tpcc --no-cpu-baseline > gpurun_out/bench32_tpcc.json 2> gpurun_out/bench32_tpcc.err
timeout 900 python bench.py --workload tpcc --loopback 4 --no-cpu-baseline > gpurun_out/bench32_tpcc_lb4.json 2> gpurun_out/bench32_tpcc_lb4.err
echo done
