mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_ycsb.py -m gpu -q -rf --timeout 300 -k "pipeline or prepare or prepared or event_log or key_not_found or search_index or dense" > gpurun_out/t2.log 2>&1; echo "t2 rc=$?"; tail -3 gpurun_out/t2.log
for f in 0 0x200; do
  timeout 600 python tools/probe_tpcc.py --W 1 --schemes tpl_nw,tpl_wd,silo,tictoc,to --lanes 32 --flags $f --watchdog 20 --reps 2 >> gpurun_out/tpcc_w1.log 2>&1
done
timeout 600 python tools/probe_tpcc.py --W 1 --schemes tpl_nw --lanes 1 --bs 32 --flags 0 --watchdog 20 --reps 2 >> gpurun_out/tpcc_w1.log 2>&1
timeout 600 python tools/probe.py --thetas 0.6,0.9 --lanes 16 --reps 3 --schemes tpl_nw,tpl_wd,silo,tictoc --flags 0x200 > gpurun_out/probe_flat.log 2>&1
timeout 600 python tools/probe.py --thetas 0.6,0.9 --lanes 16 --reps 3 --schemes tpl_nw,tpl_wd,silo,tictoc > gpurun_out/probe_scaled.log 2>&1
echo done
