mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export GCCTB_LIB=$PWD/variants/trace.so
timeout 600 python tools/trace_tail.py --schemes tpl_nw,tpl_wd,to,mvcc,silo,tictoc,gputx,gacco --thetas 0,0.6 --bucket_ns 5000 > gpurun_out/s3_trace.jsonl 2>&1
timeout 600 python tools/trace_tail.py --schemes tpl_nw,tpl_wd,to,mvcc,silo,tictoc --thetas 0.8 --bucket_ns 20000 >> gpurun_out/s3_trace.jsonl 2>&1
cut -c1-300 gpurun_out/s3_trace.jsonl
