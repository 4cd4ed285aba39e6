# K1 "what-if" timing: ncu duration / LSU pipe / issue of K1 on C3 for the in-tree library and every
# _variants/*/ build (variants may compute wrong results: timing upper bounds only)
cd "$(dirname "$0")/.."
for v in paper_1710_07745_b200 _variants/*/; do
  n=$(basename $v)
  EF_LIB_OVERRIDE=$v/libedgeforge_b200.so ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:k1v3 -s 2 -c 2 --csv --log-file gpurun_out/whatif_$n.csv python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
  python - "$n" <<'P'
import csv, sys
n = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/whatif_{n}.csv")) if len(r) > 10 and "k1v3" in r[4]]
out = {}
for r in rows:
    out.setdefault(r[-3], []).append(r[-1])
print(n, {k.split(".")[0][-28:]: v for k, v in out.items()})
P
done
