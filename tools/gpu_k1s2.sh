python -c "from oracle import oracle as O; O.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream_classifier or configs_match" > gpurun_out/t_s1.log 2>&1; echo "STREAM TESTS: $(tail -1 gpurun_out/t_s1.log)"
grep -E "^E .*AssertionError: \(" gpurun_out/t_s1.log | head -5
python bench.py --no-e2e --no-cpu --no-extra --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:k1s -s 1 -c 1 -o gpurun_out/prof_k1s python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/ncu_k1s.log 2>&1; echo ncu=$?
