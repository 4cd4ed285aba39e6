set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/t_v16.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_v16.log)"
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_v16.jsonl 2> gpurun_out/bench_v16.err; echo "BENCH rc=$?"; tail -1 gpurun_out/bench_v16.jsonl
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.jsonl 2>gpurun_out/bench_ref.err; echo "REF rc=$?"; tail -1 gpurun_out/bench_ref.jsonl
bash tools/configs_sweep.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_v16.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k1v3 -c 4 --csv --log-file gpurun_out/k1_dram_v16.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:"k1v3|hyst_local_warp" -s 2 -c 2 -o gpurun_out/prof_v16 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu3=$?
