# hysteresis iteration: suite subset first, then C3 / C1 device bench, launch lists
python -m paper_1710_07745_b200.build > /dev/null || { echo BUILD FAILED; exit 1; }
python -c "from oracle import oracle as O; O.build()" > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_h.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_h.log)"
grep -E "^E " gpurun_out/t_h.log | head -5
python bench.py --no-e2e --no-cpu > gpurun_out/b_h.log 2>&1; echo "C3 $(tail -1 gpurun_out/b_h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["extra"]["c1"]["value"], d["extra"]["c1"]["ms_per_step"], d["extra"]["c4_bands"]["value"])')"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_h_c1.csv python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu=$?
