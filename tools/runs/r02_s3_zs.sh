export PYTHONUNBUFFERED=1
B="python bench.py --steps 20 --warmup 5 --no-tpcc --no-cpu-baseline --no-index-binary --no-ceilings"
for r in 1 2; do for v in main zsmall ztiny; do
  if [ $v = main ]; then unset GCCTB_LIB; else export GCCTB_LIB=$PWD/variants/$v.so; fi
  $B > gpurun_out/zs_$v$r.json 2>/dev/null; echo "$v $(python tools/bsum.py gpurun_out/zs_$v$r.json 2>/dev/null | head -1)"
done; done
