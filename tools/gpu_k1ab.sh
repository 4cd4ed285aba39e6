# K1 A/B: parity of the in-tree build on the K1-heavy tests, then device bench
# of the in-tree library against every _variants/*/ build (interleaved twice)
python -m paper_1710_07745_b200.build > /dev/null && python -c "from oracle import oracle as O; O.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -x -q --timeout 600 -k "fast_path or configs or full or stages or dense or overflow or host or C3 or config3" > gpurun_out/t_k1.log 2>&1; echo "K1 TESTS: $(tail -1 gpurun_out/t_k1.log)"
bash tools/bench_variants.sh --no-extra "$@"
