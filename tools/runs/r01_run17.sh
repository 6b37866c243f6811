mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests17.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; tail -1 gpurun_out/smoke8.log
timeout 600 python bench.py > gpurun_out/bench17.log 2>&1
timeout 900 python bench.py --workload tpcc > gpurun_out/bench17_tpcc.log 2>&1
timeout 900 python bench.py --workload tpcc --loopback 4 > gpurun_out/bench17_tpcc_lb4.log 2>&1
timeout 900 python bench.py --workload tpcc --loopback 4 --two-pc --schemes tpl_nw,tpl_wd --no-cpu-baseline > gpurun_out/bench17_tpcc_lb4_2pc.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches17.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch17.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/prof_final2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full17.log 2>&1
timeout 900 python tools/sweep.py stages --index binary --out gpurun_out/sweep_stages_binary17.jsonl 2>&1 | tail -1
timeout 900 python tools/sweep.py stages --index dense --out gpurun_out/sweep_stages_dense17.jsonl 2>&1 | tail -1
timeout 900 python tools/sweep.py latch --out gpurun_out/sweep_latch17.jsonl 2>&1 | tail -1
timeout 1500 python tools/sweep.py theta --out gpurun_out/sweep_theta17.jsonl 2>&1 | tail -1
timeout 900 python tools/sweep.py presets --out gpurun_out/sweep_presets17.jsonl 2>&1 | tail -1
echo done
