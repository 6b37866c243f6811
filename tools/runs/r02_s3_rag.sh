mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_ycsb.py -m gpu -q --timeout 900 -k "ragged or extreme or all_writes or c1_parity" 2>&1 | tail -3
timeout 900 python tools/probe.py --reps 3 --schemes tpl_nw,tpl_wd,silo,tictoc --thetas 0.6,0.8,0.99 --lanes 16 --bs 16 --grid 148 --watchdog 60 2>&1 | cut -c1-330 > gpurun_out/s3_rag_probe.log
for v in toseq2 toseq6; do export GCCTB_LIB=$PWD/variants/$v.so; echo "# $v"; timeout 900 python tools/probe_hc.py --thetas 0.6,0.9,0.99 --schemes to --tag $v 2>&1 | cut -c1-200; done >> gpurun_out/s3_rag_probe.log
unset GCCTB_LIB
cat gpurun_out/s3_rag_probe.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l[:l.index(', \"ms_total_min')]+'}') if 'ms_total_min' in l else json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['scheme'], d['theta'], d.get('lanes', d.get('mode')), round(d['txn_s']/1e6,3), round(d['abort_rate'],2))
"
