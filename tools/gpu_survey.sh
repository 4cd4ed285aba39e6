# current per-config values and launch lists (C0, C2, C3), one full ncu capture of H1 on C3 and K1 on C2
bash tools/configs_sweep.sh
for c in 0 2 3; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo ncu_c$c=$?
done
python tools/launch_summary.py gpurun_out/launches_c0.csv gpurun_out/launches_c2.csv gpurun_out/launches_c3.csv
ncu --set full --clock-control none --import-source on -k regex:"hyst_local_warp" -s 1 -c 1 -o gpurun_out/prof_h1_c3 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/ncu_h1.log 2>&1; echo ncu_h1=$?
ncu --set full --clock-control none --import-source on -k regex:"k1v3" -s 1 -c 1 -o gpurun_out/prof_k1_c2 python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/ncu_k1c2.log 2>&1; echo ncu_k1c2=$?
