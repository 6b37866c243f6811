export PYTHONUNBUFFERED=1
for bs in 20 24 32; do
timeout 600 python tools/probe.py --reps 3 --seeds 3,4 --schemes gputx --thetas 0.6 --lanes 32 --bs $bs --grid 148 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['scheme'], d['bs'], d['seed'], 'exec', round(d['ms_exec_median'],3))
"; done
