export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -1
for r in 1 2; do
GCCTB_LIB=$PWD/variants/trace.so timeout 600 python tools/trace_kset.py --thetas 0.6,0.8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['theta'], d['ksets'], round(d['exec_ms'],3), 'detect', round(d['detect_med_us'],2), 'work', round(d['work_med_us'],2), round(d['work_p90_us'],2), 'k0', round(d['done0_us'],1))
"; done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -k "gputx" 2>&1 | tail -2
