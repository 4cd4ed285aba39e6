# peer-halo bands with the interprocess-event handshake; negative control without the waits
python -m pytest tests/test_peer_bands.py -x -q > gpurun_out/t_peer.log 2>&1; echo "PEER: $(tail -1 gpurun_out/t_peer.log)"
EF_TEST_PEER_NO_WAIT=1 python -m pytest tests/test_peer_bands.py -q -k "match_whole" > gpurun_out/t_peer_nowait.log 2>&1; echo "PEER without waits (negative control, failures expected in the delayed cases): $(tail -1 gpurun_out/t_peer_nowait.log)"
grep -E "PASSED|FAILED|passed|failed" gpurun_out/t_peer_nowait.log | tail -8
