# C3 e2e (labels + final) over unpack threads x largest chunk (MB): median ms of 40 calls each
cd "$(dirname "$0")/.."
for mb in 16 32 64; do for t in 3 4 5; do
  echo -n "chunk_mb $mb threads $t: "; EF_HOST_CHUNK_MB=$mb EF_HOST_UNPACK_THREADS=$t python tools/e2e_outliers.py 40 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["median_ms"], d["mean_ms"])'
done; done
