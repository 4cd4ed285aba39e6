# round-end style check at HEAD: GPU suite, smoke, default bench, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/t_verify.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_verify.log)"
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_verify.jsonl 2> gpurun_out/bench_verify.err; echo "BENCH rc=$?"; tail -1 gpurun_out/bench_verify.jsonl
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.jsonl 2>gpurun_out/bench_ref.err; echo "REF rc=$?"; tail -1 gpurun_out/bench_ref.jsonl
