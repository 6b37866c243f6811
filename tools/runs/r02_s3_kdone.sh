mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in main kdone0 main kdone0; do
  if [ $v = main ]; then unset GCCTB_LIB; else export GCCTB_LIB=$PWD/variants/$v.so; fi
  echo "# $v"
  timeout 600 python tools/probe.py --reps 3 --schemes gputx --thetas 0,0.6,0.8 --lanes 16 --bs 8 --grid 148 2>&1 | cut -c1-330
done > gpurun_out/s3_kdone.log
unset GCCTB_LIB
cat gpurun_out/s3_kdone.log
timeout 900 python -m pytest tests -m gpu -q -x -k gputx --timeout 600 > gpurun_out/s3k_tests.log 2>&1; tail -3 gpurun_out/s3k_tests.log
echo done
