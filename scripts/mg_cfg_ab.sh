#!/bin/bash
# A/B under the box's own (power-capped) clocks: MG solve with the k-split configs
# (TPMG_KSPLIT unset = 4x4 default, 1, 3) and programmatic dependent launch (TPMG_PDL=1),
# alternated twice.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
  for v in def ks1 ks3 pdl; do
    case $v in
      def) E="" ;; ks1) E="TPMG_KSPLIT=1" ;; ks3) E="TPMG_KSPLIT=3" ;; pdl) E="TPMG_PDL=1" ;;
    esac
    env $E timeout 300 python bench.py --solver mg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/mgab_${v}_${rep}.log 2>&1
  done
done
