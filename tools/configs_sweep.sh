# Every BASELINE config through bench.py (device-resident value, no e2e / CPU legs),
# plus radius 5 (the reference's default kernel) on C1.
for c in 0 2 3 4; do
  python bench.py --config $c --no-e2e --no-cpu > gpurun_out/cfg$c.log 2>&1
  echo "C$c rc=$? $(tail -1 gpurun_out/cfg$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], d.get("stats"))')"
done
python bench.py --radius 5 --no-e2e --no-cpu > gpurun_out/cfg1r5.log 2>&1
echo "C1 r5 rc=$? $(tail -1 gpurun_out/cfg1r5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["unit"], d["ms_per_step"], "frac", d["roofline"]["frac"], d.get("stats"))')"
