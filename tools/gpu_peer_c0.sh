python -m paper_1710_07745_b200.build > /dev/null
timeout 600 python -m pytest tests/test_peer_bands.py -x -q > gpurun_out/t_peer.log 2>&1; echo "PEER: $(tail -2 gpurun_out/t_peer.log)"
python bench.py --config 0 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/c0.jsonl 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c0.csv python bench.py --config 0 --steps 2 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu=$?
tail -1 gpurun_out/c0.jsonl | cut -c1-300
