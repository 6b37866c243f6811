# r02 session 3: launch list + ncu --set full of the eight exec launches, current code
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CMD="python bench.py --steps 2 --warmup 3 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD > gpurun_out/s3n_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_launches.csv $CMD > gpurun_out/s3n_ncu_list.log 2>&1
echo "list rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD2 > gpurun_out/s3n_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/s3n_prof $CMD2 > gpurun_out/s3n_ncu_full.log 2>&1
echo "full rc=$?"
ls -la gpurun_out/s3n_prof.ncu-rep
