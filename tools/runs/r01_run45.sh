# ncu --set full of the eight exec_tile launches of the default bench (adaptive pacing build)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/prof_v45 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_v45.log 2>&1
ls -la gpurun_out/prof_v45.ncu-rep
