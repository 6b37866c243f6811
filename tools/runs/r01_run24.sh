# GaccO hand-off idiom: relaxed polls + fence vs acquire polls; spin cap; ring microbenchmark
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "
from paper_2406_10158_b200.api import DB
db=DB(0)
for i in range(3): print(db.roofline_probe())
" > gpurun_out/roof3.log 2>&1
for v in "0 32" "1 32" "0 0" "1 0" "0 128"; do
  set -- $v
  GCCTB_NVCC_EXTRA="-DGC_GACCO_ACQ=$1 -DGC_GACCO_SPIN=$2" python -m paper_2406_10158_b200.build -f > /dev/null
  echo "# acq=$1 spin=$2"
  timeout 300 python tools/probe.py --reps 3 --schemes gacco --thetas 0.6,0.8 --lanes 16 --grid 148 --bs 24 --seeds 3,5
done > gpurun_out/gacco_poll.log 2>&1
python -m paper_2406_10158_b200.build -f > /dev/null
echo done
