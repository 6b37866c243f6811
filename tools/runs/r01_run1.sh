set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
timeout 600 python tools/probe.py --thetas 0,0.6,0.9 --lanes 16 --index dense --reps 5 > gpurun_out/probe_dense.log 2>&1
timeout 600 python tools/probe.py --thetas 0,0.6,0.9 --lanes 16 --index tree --reps 5 > gpurun_out/probe_tree.log 2>&1
timeout 600 python tools/probe.py --thetas 0,0.6 --lanes 16 --index dense --reps 5 --chunk 4 > gpurun_out/probe_chunk4.log 2>&1
timeout 600 python tools/probe.py --thetas 0,0.6 --lanes 1 --index dense --reps 3 > gpurun_out/probe_thread_dense.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --index tree > gpurun_out/bench_tree.log 2>&1
timeout 900 python bench.py --workload tpcc --loopback 4 > gpurun_out/bench_tpcc_lb4.log 2>&1
timeout 900 python bench.py --workload tpcc > gpurun_out/bench_tpcc.log 2>&1
echo done
