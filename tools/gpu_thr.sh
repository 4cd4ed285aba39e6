# H1 path threshold A/B on the one-frame configs (device bench)
for c in 0 2; do for thr in 32 8 0; do
  EF_H1_BLOCK_TILES_PER_SM=$thr python bench.py --config $c --no-e2e --no-cpu --no-extra > gpurun_out/thr.log 2>&1
  echo "C$c thr=$thr $(tail -1 gpurun_out/thr.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done; done
for c in 0 2; do ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_thr0_c$c.csv env EF_H1_BLOCK_TILES_PER_SM=0 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; done
