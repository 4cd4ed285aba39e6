for i in 1 2 3; do
python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('full', e['ms_per_step'], e['step_ms_rank0']['all'], e['edges_only']['step_ms_rank0']['all'])"
done
