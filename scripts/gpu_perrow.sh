#!/bin/bash
# 1 GPU: per-level MG kernel times with the k-split in-place boxes loaded row by row for every
# tile (TPMG_DBG_PERROW=1) vs as one box (default), to price the strip-boundary path.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-pr}
export TPMG_PROF_DETAIL=1
for v in "" "TPMG_DBG_PERROW=1"; do
  env $v timeout 300 python bench.py --solver mg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/det_${TAG}_${#v}.json 2> gpurun_out/det_${TAG}_${#v}.err
done
