mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/tb_bench.json 2> gpurun_out/tb_bench.err; python tools/bsum.py gpurun_out/tb_bench.json 2>/dev/null | head -1; tail -2 gpurun_out/tb_bench.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/tb_bench.json').read().strip().splitlines()[-1])
for k,v in d['tpcc'].items():
    print(k, round(v['value']/1e6,2), {s:(round(x['txn_s']/1e6,2), round(x['abort_rate'],2)) for s,x in v['per_scheme'].items()})
P
timeout 2400 python -m pytest tests/test_gpu_tpcc.py tests/test_gpu_c4.py -m gpu -q --timeout 900 -k "bench_launch" > gpurun_out/tb_tests.log 2>&1; tail -2 gpurun_out/tb_tests.log
