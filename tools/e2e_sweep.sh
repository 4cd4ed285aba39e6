#!/bin/bash
# sweep of the host pipeline's tunables (run on the GPU box)
out=gpurun_out/e2e_sweep.log; : > $out
for rep in 1 2; do for t in 2 3 4; do for c in 4 6 8 12; do
  echo "threads=$t chunkMB=$c $(EF_HOST_UNPACK_THREADS=$t EF_HOST_CHUNK_MB=$c python tools/e2e_probe.py 2>&1 | grep 'host pinned')" >> $out
done; done; done
