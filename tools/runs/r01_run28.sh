# f-3 Eytzinger index: parity tests, then the Exp-6 stage sweep per index method
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q -k "index" > gpurun_out/t28.log 2>&1; tail -1 gpurun_out/t28.log
for ix in dense tree binary eytz; do
  timeout 600 python tools/sweep.py stages --index $ix --out gpurun_out/stages_$ix.jsonl 2>> gpurun_out/stages28.err
done
for ix in dense tree binary eytz; do
  timeout 300 python tools/probe.py --reps 3 --thetas 0 --W 0 --lanes 16 --grid 148 --bs 16 --index $ix --schemes tpl_nw,silo,gacco
done > gpurun_out/index_ro.log 2>&1
echo done
