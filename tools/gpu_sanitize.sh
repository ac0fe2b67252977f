# usage: bash tools/gpu_sanitize.sh <tool>   (one compute-sanitizer tool per call; B200_PROFILING.md)
T=${1:-memcheck}
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $T --error-exitcode 99 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/sanitize_plain.log; tail -25 gpurun_out/sanitize_$T.log
