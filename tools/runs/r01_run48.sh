# re-tune warps per SM for GaccO / GPUTx (exec time; a3 is pipelined in the bench)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for bs in 16 20 24 32; do
  timeout 300 python tools/probe.py --reps 5 --schemes gacco --thetas 0.6 --seeds 3,5 --lanes 16 --grid 148 --bs $bs > gpurun_out/tune48_gacco_bs$bs.log 2>&1
done
for bs in 4 6 8 12 16; do
  timeout 300 python tools/probe.py --reps 5 --schemes gputx --thetas 0.6 --seeds 3,5 --lanes 16 --grid 148 --bs $bs > gpurun_out/tune48_gputx_bs$bs.log 2>&1
done
echo done
