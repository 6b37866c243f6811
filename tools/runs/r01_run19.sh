# occupancy experiment: executor launch bounds (registers vs resident transactions)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,to,mvcc,silo,tictoc,gputx,gacco
python -m paper_2406_10158_b200.build -f > /dev/null
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 16 --bs 32 > gpurun_out/occ_1024x1.log 2>&1
for v in "512 3 16" "448 3 14" "512 4 16"; do
  set -- $v
  GCCTB_NVCC_EXTRA="-DGC_EXEC_MAXT=$1 -DGC_EXEC_MINB=$2" python -m paper_2406_10158_b200.build -f > /dev/null
  timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 16 --bs $3 > gpurun_out/occ_${1}x${2}.log 2>&1
done
python -m paper_2406_10158_b200.build -f > /dev/null
echo done
