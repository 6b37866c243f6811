mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in trace nwi2 nwi8; do
  export GCCTB_LIB=$PWD/variants/$v.so
  echo "# $v"
  timeout 600 python tools/trace_tail.py --schemes tpl_nw --thetas 0.6 --bucket_ns 5000 2>&1 | cut -c1-260
  timeout 600 python tools/trace_tail.py --schemes tpl_nw --thetas 0.6 --bucket_ns 5000 2>&1 | cut -c1-260
  timeout 600 python tools/trace_tail.py --schemes tpl_nw --thetas 0.8,0.9 --bucket_ns 20000 2>&1 | cut -c1-260
done > gpurun_out/s3_nwi.log
cat gpurun_out/s3_nwi.log
