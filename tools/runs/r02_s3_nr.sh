export PYTHONUNBUFFERED=1
for v in trace noread; do echo "# $v"; for r in 1 2; do
GCCTB_LIB=$PWD/variants/$v.so timeout 600 python tools/trace_kset.py --thetas 0.6,0.8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['theta'], d['ksets'], round(d['exec_ms'],3), 'detect', round(d['detect_med_us'],2), 'work', round(d['work_med_us'],2), round(d['work_p90_us'],2), 'k0', round(d['done0_us'],1))
"; done; done
