# adaptive jitter at very high contention: GC_JITTER_LO=32 (shipped) vs 0 (static cap), Silo / TicToc / 2PL, theta 0.9 / 0.99 (sweep launch: tile 16, full grid)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=silo,tictoc,tpl_nw,tpl_wd
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0.9,0.99 --seeds 3 --lanes 16 --bs 32 > gpurun_out/hc50_lo32.log 2>&1
GCCTB_NVCC_EXTRA="-DGC_JITTER_LO=0" python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0.9,0.99 --seeds 3 --lanes 16 --bs 32 > gpurun_out/hc50_lo0.log 2>&1
python -m paper_2406_10158_b200.build -f > /dev/null 2>&1
echo done
