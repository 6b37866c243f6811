mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; python tools/bsum.py gpurun_out/fin_bench.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; tail -c 400 gpurun_out/fin_ref.json
CMD="python bench.py --steps 2 --warmup 3 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD > gpurun_out/fin_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_ncu_list.log 2>&1
echo "list rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-tpcc --no-cpu-baseline --no-ceilings --no-index-binary"
$CMD2 > gpurun_out/fin_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:exec_tile_kernel -c 8 -o gpurun_out/fin_prof $CMD2 > gpurun_out/fin_ncu_full.log 2>&1
echo "full rc=$?"
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin_tests.log 2>&1; tail -3 gpurun_out/fin_tests.log
echo done
