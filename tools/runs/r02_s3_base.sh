mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/s3_smoke.log 2>&1; tail -2 gpurun_out/s3_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3_bench_base.json 2> gpurun_out/s3_bench_base.err; tail -c 600 gpurun_out/s3_bench_base.json
timeout 600 python tools/probe.py --reps 3 --schemes gacco,gputx --thetas 0,0.6,0.8 --lanes 16 > gpurun_out/s3_probe_det_base.log 2>&1; tail -20 gpurun_out/s3_probe_det_base.log
echo done
