mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for L in 16 32; do for bs in 8 16; do
timeout 600 python tools/probe.py --reps 3 --schemes gputx,gacco --thetas 0.6,0.8 --lanes $L --bs $bs --grid 148 --watchdog 60 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], 'lanes', d['lanes'], 'bs', d['bs'], 'exec', round(d['ms_exec_median'],3))
"
done; done
