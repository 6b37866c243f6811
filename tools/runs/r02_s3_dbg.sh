export PYTHONUNBUFFERED=1
for s in silo to tpl_nw; do timeout 900 python tools/dbg_2pc.py $s 60 2>&1 | tail -20; done
