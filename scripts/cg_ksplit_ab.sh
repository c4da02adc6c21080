#!/bin/bash
# A/B under the box's own (power-capped) clocks: PCG with the one-thread-per-column CGPREC
# (default) vs the k-split CGPREC (TPMG_KSPLIT_CG=1, 16 warps per SM), alternated 3 times.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2 3; do
  for ks in 0 1; do
    TPMG_KSPLIT_CG=$ks timeout 300 python bench.py --solver cg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/cgks_${ks}_${rep}.log 2>&1
  done
done
