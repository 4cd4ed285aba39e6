# C1 and C3 e2e of the in-tree library against every _variants/*/ build, interleaved
cd "$(dirname "$0")/.."
for i in 1 2 3; do
for lib in paper_1710_07745_b200 _variants/*/; do
EF_LIB_OVERRIDE=$lib/libedgeforge_b200.so python bench.py --config 1 --no-cpu --no-extra 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$lib', 'C1 e2e ms', e['ms_per_step'], 'median', e['step_ms_rank0']['median'], 'edges-only', e['edges_only']['ms_per_step'])"
done; done
for i in 1 2; do
for lib in paper_1710_07745_b200 _variants/*/; do
EF_LIB_OVERRIDE=$lib/libedgeforge_b200.so python tools/e2e_outliers.py 60
done; done
