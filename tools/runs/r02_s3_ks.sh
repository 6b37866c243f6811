mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
GCCTB_LIB=$PWD/variants/trace.so timeout 600 python tools/trace_kset.py --thetas 0.6,0.8 > gpurun_out/s3_kset.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/s3_kset.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print({k:v for k,v in d.items() if not k.endswith('_us') or not isinstance(v,list)})
    print('done', d['done_us'][:12], '...', d['done_us'][-8:])
    print('first', d['first_us'][:12], '...', d['first_us'][-8:])
"
bash tools/runs/r02_s3_tune.sh
