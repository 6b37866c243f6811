mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in main h2pl64 h2pl256; do
  if [ $v = main ]; then unset GCCTB_LIB; else export GCCTB_LIB=$PWD/variants/$v.so; fi
  echo "# $v"
  timeout 600 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --schemes tpl_nw,tpl_wd --lanes 32 --reps 3 --watchdog 60 2>&1 | cut -c1-200
  timeout 600 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --schemes tpl_nw,tpl_wd --lanes 32 --reps 3 --watchdog 60 2>&1 | cut -c1-200
done > gpurun_out/s3_tpcch.log
cat gpurun_out/s3_tpcch.log
