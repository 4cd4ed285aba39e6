# The GPU suite against the debug build (device bounds assertions, -DEF_DEBUG_CHECKS):
# the substitute for compute-sanitizer, which is closed on this pool.
#   bash tools/variants.sh debug "-DEF_DEBUG_CHECKS"   (here, before the call)
python -c "from oracle import oracle as O; O.build()"
export EF_LIB_OVERRIDE=$PWD/_variants/debug/libedgeforge_b200.so
timeout 2000 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/t_debug.log 2>&1; echo "DEBUG TESTS: $(tail -1 gpurun_out/t_debug.log)"
grep -c "EF_DCHECK failed" gpurun_out/t_debug.log
timeout 600 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/bench_debug.jsonl 2>&1; echo "bench rc=$?"; grep -c "EF_DCHECK" gpurun_out/bench_debug.jsonl
