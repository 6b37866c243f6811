export PYTHONUNBUFFERED=1
timeout 900 python bench.py --workload tpcc --warehouses 512 --loopback 4 --steps 3 --warmup 1 > gpurun_out/lb4_p2p.json 2> gpurun_out/lb4_p2p.err; tail -c 700 gpurun_out/lb4_p2p.json; tail -3 gpurun_out/lb4_p2p.err
