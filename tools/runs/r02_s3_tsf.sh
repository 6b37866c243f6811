mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in main tsf256 tsf1024; do
  if [ $v = main ]; then unset GCCTB_LIB; else export GCCTB_LIB=$PWD/variants/$v.so; fi
  echo "# $v"
  timeout 1500 python tools/probe_hc.py --thetas 0.6,0.8,0.9,0.95,0.99 --schemes to,mvcc --tag $v 2>&1 | cut -c1-200
done > gpurun_out/s3_tsf.log
python - <<'P'
import json
for l in open('gpurun_out/s3_tsf.log'):
    if l.startswith('#'): print(l.strip()); continue
    try: d=json.loads(l)
    except Exception: print(l[:150]); continue
    print(d['scheme'], d['theta'], d['mode'], round(d['txn_s']/1e6,3), round(d['abort_rate'],1))
P
