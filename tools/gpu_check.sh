# full GPU suite + smoke + default bench + C0/C2 lines
python -m paper_1710_07745_b200.build > /dev/null && python -c "from oracle import oracle as O; O.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_all.log)"
grep -E "FAILED|Error" gpurun_out/t_all.log | head -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_chk.jsonl 2> gpurun_out/bench_chk.err; echo "BENCH rc=$?"; tail -1 gpurun_out/bench_chk.jsonl | cut -c1-400
for c in 0 2; do timeout 300 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench_c$c.jsonl 2>&1; tail -1 gpurun_out/bench_c$c.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c', d['ms_per_step'], d['value'], d['stats'])"; done
