mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for bs in 8 12 16 20 24 32; do
  timeout 900 python tools/probe.py --reps 3 --seeds 3,4 --schemes tpl_nw,tpl_wd,to,mvcc,silo,tictoc,gputx,gacco --thetas 0.6 --lanes 16 --bs $bs --grid 148 --watchdog 60 2>&1
done > gpurun_out/s3_tune.log
python - <<'P'
import json, collections
t = collections.defaultdict(dict)
for l in open('gpurun_out/s3_tune.log'):
    try: d = json.loads(l)
    except Exception: continue
    t[d['scheme']].setdefault(d['bs'], []).append(d['ms_exec_median'] if 'ms_exec_median' in d else d['ms_total_median'])
for s, v in t.items():
    print(s, {bs: round(sum(x)/len(x), 3) for bs, x in sorted(v.items())})
P
