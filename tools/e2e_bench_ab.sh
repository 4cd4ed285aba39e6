for i in 1 2 3; do
for lib in paper_1710_07745_b200 _variants/blocksync; do
EF_LIB_OVERRIDE=$lib/libedgeforge_b200.so python bench.py --no-cpu --no-extra 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$lib', e['ms_per_step'], e['step_ms_rank0']['all'], e['edges_only']['step_ms_rank0']['max'])"
done; done
