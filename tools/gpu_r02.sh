# round-2 GPU pass: tests, smoke, bench (C3 headline), reference arm, launch list,
# K1 DRAM bytes on C3, one --set full capture of K1 on C3.
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_1710_07745_b200.build > /dev/null || { echo BUILD FAILED; exit 1; }
python -c "from oracle import oracle as O; O.build()"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/t_$T.log 2>&1; echo "TESTS: $(tail -1 gpurun_out/t_$T.log)"
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log
python bench.py > gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_$T.err; echo "BENCH rc=$?"; tail -1 gpurun_out/bench_$T.jsonl
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$T.jsonl 2>gpurun_out/bench_ref_$T.err; echo "REF rc=$?"; tail -1 gpurun_out/bench_ref_$T.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu1=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k1v3 -c 4 --csv --log-file gpurun_out/k1_dram_c3_$T.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu2=$?
if [ -z "$NO_FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:"k1v3" -s 1 -c 1 -o gpurun_out/prof_k1_$T python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/ncu_full_$T.log 2>&1; echo ncu3=$?
fi
