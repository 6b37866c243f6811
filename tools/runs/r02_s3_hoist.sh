mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/s3h_smoke.log 2>&1; tail -2 gpurun_out/s3h_smoke.log
timeout 900 python -m pytest tests -m gpu -q -x -k gacco --timeout 600 > gpurun_out/s3h_tests.log 2>&1; tail -3 gpurun_out/s3h_tests.log
timeout 600 python tools/probe.py --reps 3 --schemes gacco --thetas 0,0.6,0.8 --lanes 16 > gpurun_out/s3h_probe.log 2>&1; cat gpurun_out/s3h_probe.log | cut -c1-400
timeout 600 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6 --lanes 1 --wd 5 --bs 8 > gpurun_out/s3h_probe_thread.log 2>&1; tail -2 gpurun_out/s3h_probe_thread.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3h_bench.json 2> gpurun_out/s3h_bench.err; tail -c 300 gpurun_out/s3h_bench.json
echo done
