# quick K1 iteration: GPU parity tests + device-resident bench (no e2e / CPU legs) + K1 launch times
python -m pytest tests -m gpu -x -q > gpurun_out/t_q.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_q.log)"
for i in 1 2; do python bench.py --no-e2e --no-cpu > gpurun_out/b_q$i.log 2>&1; echo "BENCH$i rc=$? $(tail -1 gpurun_out/b_q$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"])')"; done
