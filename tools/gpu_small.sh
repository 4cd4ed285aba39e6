# launch lists of the single-frame configs (C0 512^2, C2 4096^2)
python -m paper_1710_07745_b200.build > /dev/null
for c in 0 2; do
python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/plain_c$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 8 -c 16 --csv --log-file gpurun_out/launches_c${c}_r02.csv python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu c$c=$?"
done
