# C3 e2e (labels + final, and edges only) by the number of host threads that unpack a chunk
# while later chunks are still copying (EF_HOST_UNPACK_THREADS; the last chunk uses the whole pool)
cd "$(dirname "$0")/.."
for t in 2 3 4 6 8 12 16; do
  EF_HOST_UNPACK_THREADS=$t python bench.py --steps 5 --warmup 3 --no-cpu --no-extra 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read()); e=d["e2e"]
print("threads", '$t', "e2e ms", e["ms_per_step"], "median", e["step_ms_rank0"]["median"], "edges-only ms", e["edges_only"]["ms_per_step"], "median", e["edges_only"]["step_ms_rank0"]["median"])'
done
