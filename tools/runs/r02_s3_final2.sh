mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin2_smoke.log 2>&1; tail -1 gpurun_out/fin2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err; python tools/bsum.py gpurun_out/fin2_bench.json 2>/dev/null
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin2_tests.log 2>&1; tail -3 gpurun_out/fin2_tests.log
timeout 1500 python tools/probe_hc.py --thetas 0.6,0.8,0.9,0.95,0.99 --tag final > gpurun_out/fin2_hc.jsonl 2>&1; tail -1 gpurun_out/fin2_hc.jsonl
echo done
