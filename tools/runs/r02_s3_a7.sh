mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 --no-tpcc --no-cpu-baseline > gpurun_out/a7_bench.json 2> gpurun_out/a7_bench.err; python tools/bsum.py gpurun_out/a7_bench.json 2>/dev/null
timeout 2400 python -m pytest tests/test_gpu_ycsb.py tests/test_gpu_partition.py tests/test_gpu_pipeline.py -m gpu -q --timeout 900 -x 2>&1 | tail -2
