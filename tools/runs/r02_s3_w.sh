mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export GCCTB_LIB=$PWD/variants/trace.so
for w in 0.0 0.02 0.1 0.3; do
  timeout 600 python tools/trace_tail.py --schemes tpl_nw,silo,to,mvcc --thetas 0.6 --W $w --bucket_ns 5000 2>&1 | cut -c1-230
done > gpurun_out/s3_w.log
timeout 600 python tools/trace_tail.py --schemes tpl_nw,silo --thetas 0.3,0.5,0.7 --bucket_ns 5000 2>&1 | cut -c1-230 >> gpurun_out/s3_w.log
cat gpurun_out/s3_w.log
