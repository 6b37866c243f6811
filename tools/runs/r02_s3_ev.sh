export PYTHONUNBUFFERED=1
B="python bench.py --steps 20 --warmup 5 --no-tpcc --no-cpu-baseline --no-index-binary --no-ceilings"
for r in 1 2; do
  for o in "" "--no-phase-events" "--no-phase-events --no-scheme-events"; do
    $B $o > gpurun_out/ev.json 2>gpurun_out/ev.err; python -c "
import json; d=json.loads(open('gpurun_out/ev.json').read().strip().splitlines()[-1]); print('$o', round(d['value']/1e6,2), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1))" || tail -3 gpurun_out/ev.err
  done
done
