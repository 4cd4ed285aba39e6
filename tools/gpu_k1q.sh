# K1 change check: GPU parity suite, C3 / C2 / C1 device values, K1 launch times
python -m pytest tests -m gpu -x -q > gpurun_out/t_q.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_q.log)"
for c in 3 2 1; do for i in 1 2; do python bench.py --config $c --no-e2e --no-cpu --no-extra > gpurun_out/b_q$c$i.log 2>&1; echo "C$c/$i rc=$? $(tail -1 gpurun_out/b_q$c$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"; done; done
for c in 3 2; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/lq_c$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
done
python tools/launch_summary.py gpurun_out/lq_c3.csv gpurun_out/lq_c2.csv
