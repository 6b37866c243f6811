# launch list + ncu --set full of the 8 exec launches (current code, tuned launch)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches26.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch26.log 2>&1
python tools/launch_summary.py gpurun_out/launches26.csv > gpurun_out/launches26.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/prof26 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full26.log 2>&1
CFG=$(python -c "import sys; sys.argv=['bench.py']; import bench; print(bench.config_key(bench.parse()))")
echo "cfg=$CFG"
python tools/ncu_summary.py gpurun_out/prof26.ncu-rep gpurun_out/r01_ncu_exec_tile_v20.md --config "$CFG" --title "exec_tile_kernel, YCSB configs[1] (MC), tile 16, tuned launch, acquire-poll hand-offs" > /dev/null 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic26.json
ls -la gpurun_out/prof26.ncu-rep
echo done
