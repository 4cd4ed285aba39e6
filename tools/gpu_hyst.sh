# hysteresis iteration: full GPU suite, configs sweep (device value), C3 launch list
python -m paper_1710_07745_b200.build > /dev/null && python -c "from oracle import oracle as O; O.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_h.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_h.log)"
bash tools/configs_sweep.sh
python bench.py --no-e2e --no-cpu --no-extra > gpurun_out/b_h.log 2>&1; echo "C3 $(tail -1 gpurun_out/b_h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["stats"])')"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu=$?
for c in 0 2; do ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_h_c$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; done
