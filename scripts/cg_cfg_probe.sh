#!/bin/bash
# CG iteration time with the k-split CG preconditioner configs vs the one-thread-per-column kernel.
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_1402_3545_b200.build > /dev/null 2>&1
for r in 1 2; do
  for ks in 0 2 1 3; do
    echo -n "TPMG_KSPLIT=$ks "
    TPMG_KSPLIT=$ks python scripts/ab_probe.py . 2>&1 | tail -1
  done
done > gpurun_out/cg_cfg.txt
