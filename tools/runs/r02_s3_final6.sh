mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin6_smoke.log 2>&1; tail -1 gpurun_out/fin6_smoke.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fin6_tests.log 2>&1; tail -3 gpurun_out/fin6_tests.log
echo done
