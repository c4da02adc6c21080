#!/bin/bash
# A/B of the k_line tile bands on wide grids: PCG at 4096^2 and 2048^2 (one GPU), band 32 vs off.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-band}
for rep in 1 2; do
  for cfg in "--global-nx 4096" "--per-gpu-nx 2048"; do
    for v in "" "TPMG_BAND=0"; do
      name=$(echo "$cfg $v" | sed 's/[ =-]//g')
      env $v timeout 600 python bench.py $cfg --solver cg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
        > gpurun_out/ab_${TAG}_${name}_${rep}.json 2> gpurun_out/ab_${TAG}_${name}_${rep}.err
    done
  done
done
