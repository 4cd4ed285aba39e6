# one compute-sanitizer tool per call (B200_PROFILING.md); the plain run first
TOOL=${1:-racecheck}
python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 && \
compute-sanitizer --tool $TOOL --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/sanitize_$TOOL.log
