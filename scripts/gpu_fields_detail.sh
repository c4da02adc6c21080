#!/bin/bash
# Per-level kernel times of the MG solve with per-column fields (TPMG_PROF_DETAIL=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-fd}
export TPMG_PROF_DETAIL=1
for v in "" "TPMG_PIVOTS=0"; do
  env $v timeout 300 python bench.py --solver mg --fields smooth --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/det_${TAG}_${#v}.json 2> gpurun_out/det_${TAG}_${#v}.err
done
timeout 300 python bench.py --solver mg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/det_${TAG}_flat.json 2> gpurun_out/det_${TAG}_flat.err
