python -m paper_1710_07745_b200.build > /dev/null && python -c "from oracle import oracle as O; O.build()"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "bit_sweep or hysteresis_vs_oracle" > gpurun_out/t_hb1.log 2>&1; echo "HB TESTS: $(tail -3 gpurun_out/t_hb1.log)"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_hb2.log 2>&1; echo "ALL: $(tail -3 gpurun_out/t_hb2.log)"
timeout 300 python bench.py --no-cpu > gpurun_out/bench_hb.jsonl 2> gpurun_out/bench_hb.err; echo "BENCH rc=$?"; tail -1 gpurun_out/bench_hb.jsonl | cut -c1-600
