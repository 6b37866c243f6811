mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,to,mvcc,silo,tictoc,gputx,gacco
( for cfg in "64 65536 5114 0x2000" "512 65536 5114 0x2000"; do set -- $cfg
  for g in 148 0; do for bs in 4 8 16; do
    timeout 900 python tools/probe_tpcc.py --W $1 --batch $2 --mix $3 --flags $4 --schemes $S --lanes 32 --bs $bs --grid $g --reps 2 --watchdog 60 2>&1
  done; done; done
  for bs in 1 2 4; do timeout 900 python tools/probe_tpcc.py --W 1 --batch 16384 --mix 5000 --schemes $S --lanes 32 --bs $bs --grid 148 --reps 2 --watchdog 60 2>&1; done
) > gpurun_out/s3_tpcctune.jsonl
python - <<'P'
import json, collections
t = collections.defaultdict(dict)
for l in open('gpurun_out/s3_tpcctune.jsonl'):
    try: d = json.loads(l)
    except Exception: continue
    t[(d['W'], d['scheme'])][(d['bs'], d['grid'])] = round(d['txn_s'] / 1e6, 2)
for k, v in sorted(t.items()):
    best = max(v, key=v.get)
    print(k, 'best', best, v[best], v)
P
