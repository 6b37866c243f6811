mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export GCCTB_LIB=$PWD/variants/trace.so
for s in tpl_nw:32 tpl_wd:32 to:16 mvcc:24 silo:24 tictoc:24 gputx:8 gacco:8; do
  sc=${s%%:*}; bs=${s##*:}
  timeout 600 python tools/trace_tail.py --schemes $sc --thetas 0.6 --lanes 32 --bs $bs --bucket_ns 5000 2>&1
done > gpurun_out/s3_tr32.jsonl
python -c "
import json
for l in open('gpurun_out/s3_tr32.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['scheme'], round(d['exec_ms'],3), d['t50_us'], d['t90_us'], d['t99_us'], d['t100_us'])
"
