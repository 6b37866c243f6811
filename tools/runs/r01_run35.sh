# f-3 metadata layout ablation: packed 8 B SoA control words (shipped) vs one word per 32 B sector
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=tpl_nw,tpl_wd,to,silo,tictoc
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6,0.8 --lanes 16 --grid 148 --bs 16 > gpurun_out/meta_packed.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 1 --bs 32 > gpurun_out/meta_packed_thread.log 2>&1
timeout 600 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs 8 --grid 148 --reps 2 --schemes $S > gpurun_out/meta_packed_tpcc.log 2>&1
GCCTB_NVCC_EXTRA="-DGC_META_STRIDE=4" python -m paper_2406_10158_b200.build -f > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q -k "test_c1_parity or brute_force or latched or w4_parity or test_c2_full_size_parity" > gpurun_out/t35_pad.log 2>&1; tail -1 gpurun_out/t35_pad.log
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6,0.8 --lanes 16 --grid 148 --bs 16 > gpurun_out/meta_pad.log 2>&1
timeout 600 python tools/probe.py --reps 3 --schemes $S --thetas 0,0.6 --lanes 1 --bs 32 > gpurun_out/meta_pad_thread.log 2>&1
timeout 600 python tools/probe_tpcc.py --W 64 --batch 65536 --mix 5114 --bs 8 --grid 148 --reps 2 --schemes $S > gpurun_out/meta_pad_tpcc.log 2>&1
python -m paper_2406_10158_b200.build -f > /dev/null
echo done
