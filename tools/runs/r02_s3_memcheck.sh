mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python tools/sanitize.py > gpurun_out/mc_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize.py > gpurun_out/r02_sanitize_memcheck_s3.txt 2>&1
echo "rc=$?"; tail -5 gpurun_out/r02_sanitize_memcheck_s3.txt
