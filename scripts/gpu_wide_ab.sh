#!/bin/bash
# A/B of PCG on wide grids: each line of $CFGS is "nx [ENV=V ...]"; one bench line per entry
# (gpurun_out/wide_${TAG}_<nx><env>.json).  scripts/wide_summary.py reads them.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-wab}
i=0
while read -r line; do
  [ -z "$line" ] && continue
  i=$((i + 1))
  set -- $line
  nx=$1; shift
  name=$(echo "$nx $*" | sed 's/[ =/.]//g;s/TPMG_//g')
  [ -n "$REPNAMES" ] && name="${name}_$i"
  env "$@" timeout 900 python bench.py --global-nx $nx --solver ${SOLVER:-cg} --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/wide_${TAG}_${name}.json 2> gpurun_out/wide_${TAG}_${name}.err
done <<< "$CFGS"
