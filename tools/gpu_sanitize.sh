# one compute-sanitizer tool per gpurun call (B200_PROFILING.md); usage: bash tools/gpu_sanitize.sh <tool>
T=${1:-memcheck}
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$T.log 2>&1
echo "exit $?"; tail -8 gpurun_out/r02_sanitize_$T.log
