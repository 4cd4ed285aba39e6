# streaming classifier iteration: its parity tests first, then the suite, then device bench A/B
python -c "from oracle import oracle as O; O.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream_classifier or configs_match" > gpurun_out/t_s1.log 2>&1; echo "STREAM TESTS: $(tail -1 gpurun_out/t_s1.log)"
grep -E "^E |Error|error" gpurun_out/t_s1.log | head -20
one() {  # name libpath envs...
  env "${@:3}" EF_LIB_OVERRIDE=$2 python bench.py --no-e2e --no-cpu --no-extra 2>gpurun_out/err_$1.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$1'", d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"], d["stats"]["fixups"])'
}
for rep in 1 2; do
  one stream paper_1710_07745_b200/libedgeforge_b200.so
  one tile paper_1710_07745_b200/libedgeforge_b200.so EF_K1_VARIANT=0
  one minb5 _variants/minb5/libedgeforge_b200.so
  one seg128 paper_1710_07745_b200/libedgeforge_b200.so EF_K1S_SEG=128
  one seg32 paper_1710_07745_b200/libedgeforge_b200.so EF_K1S_SEG=32
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_s2.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_s2.log)"
