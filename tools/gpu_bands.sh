# band path: device seam merge parity + C4 band bench at N=1
python -m pytest tests -m gpu -x -q -k "band or merge" > gpurun_out/t_bands.log 2>&1; echo "BAND TESTS: $(tail -1 gpurun_out/t_bands.log)"
python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "ALL TESTS: $(tail -1 gpurun_out/t_all.log)"
python bench.py --config 4 --bands --steps 10 --warmup 3 > gpurun_out/bands_c4.log 2>&1; echo "C4 bands rc=$?"; tail -2 gpurun_out/bands_c4.log
