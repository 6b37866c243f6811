mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin5_smoke.log 2>&1; tail -1 gpurun_out/fin5_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin5_bench.json 2> gpurun_out/fin5_bench.err; python tools/bsum.py gpurun_out/fin5_bench.json 2>/dev/null | head -1; tail -2 gpurun_out/fin5_bench.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin5_bench2.json 2> /dev/null; python tools/bsum.py gpurun_out/fin5_bench2.json 2>/dev/null | head -1
timeout 2400 python -m pytest tests/test_gpu_ycsb.py tests/test_gpu_tpcc.py -m gpu -q --timeout 900 -x 2>&1 | tail -1
