mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/probe.py --reps 2 --watchdog 60 --schemes to --thetas 0.6,0.8,0.9,0.95,0.99 --lanes 16 > gpurun_out/to_v10.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes mvcc,to --thetas 0,0.6,0.9 --lanes 16 > gpurun_out/mvcc_inter.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes mvcc --thetas 0,0.6,0.9 --lanes 16 --flags 0x400 > gpurun_out/mvcc_split.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes mvcc,to --thetas 0,0.6 --lanes 1 > gpurun_out/mvcc_inter_thread.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes mvcc --thetas 0,0.6 --lanes 1 --flags 0x400 > gpurun_out/mvcc_split_thread.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -k "to- or to] or mvcc or ts_overflow" > gpurun_out/t10.log 2>&1; tail -3 gpurun_out/t10.log
echo done
