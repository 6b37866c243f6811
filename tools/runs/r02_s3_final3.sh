mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin3_bench.json 2> gpurun_out/fin3_bench.err; python tools/bsum.py gpurun_out/fin3_bench.json 2>/dev/null | head -1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin3_ref.json 2> gpurun_out/fin3_ref.err; tail -c 200 gpurun_out/fin3_ref.json
CMD="python bench.py --steps 2 --warmup 3 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD > gpurun_out/fin3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin3_launches.csv $CMD > gpurun_out/fin3_ncu_list.log 2>&1
echo "list rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD2 > gpurun_out/fin3_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/fin3_prof $CMD2 > gpurun_out/fin3_ncu_full.log 2>&1
echo "full rc=$?"
