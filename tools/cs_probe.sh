set -x
ls -la /usr/local/cuda/bin/compute-sanitizer
/usr/local/cuda/bin/compute-sanitizer --version 2>&1 | head -3
CUDA_LAUNCH_BLOCKING=0 timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py p1_128 2>&1 | tail -15
echo rc=$?
