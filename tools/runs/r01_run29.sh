mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "silo or verify or events" > gpurun_out/t29.log 2>&1; tail -1 gpurun_out/t29.log
for ix in dense binary; do
  timeout 600 python tools/sweep.py stages --index $ix --out gpurun_out/stages29_$ix.jsonl 2>> gpurun_out/stages29.err
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench29.json 2> gpurun_out/bench29.err
echo done
