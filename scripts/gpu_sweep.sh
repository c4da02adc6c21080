#!/bin/bash
# Parameter sweeps on one B200 (supplementary bench lines, not the headline):
#   C3  - nu_CFL sweep {2, 4, 6, 8.4, 10} at 1024^2 x 128, MG and PCG
#   ROB - sec:Robustness schedules: L in {5, 7, 10} x nu in {8.4, 84, 840} with the paper's
#         coarse-sweep counts, MG only, face-Dirichlet boundary [R25]
#   C5  - 4096^2 x 128 (2^31 unknowns) on one GPU, MG and PCG (strong-scaling base point)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
OUT=gpurun_out/sweep_$TAG.jsonl
[ -n "$APPEND" ] || : > $OUT
run() {
  timeout 600 python bench.py --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/sweep_one.log 2>&1
  rc=$?
  if [ $rc -eq 0 ]; then grep '^{' gpurun_out/sweep_one.log | tail -1 >> $OUT; else echo "{\"failed\": \"$*\", \"rc\": $rc}" >> $OUT; tail -5 gpurun_out/sweep_one.log >> gpurun_out/sweep_err_$TAG.log; fi
}
if [ -z "$ONLY" ] || [ "$ONLY" = c3 ]; then
  for nu in 2 4 6 8.4 10; do run --nu $nu; done
fi
if [ -z "$ONLY" ] || [ "$ONLY" = rob ]; then
  for spec in "5 8.4 2" "5 16.8 2" "5 84 30" "5 840 150" "7 8.4 2" "7 84 5" "7 840 15" "10 8.4 2" "10 84 2" "10 840 2"; do
    set -- $spec
    run --solver mg --levels $1 --nu $2 --coarse-sweeps $3 --boundary 1
  done
fi
if [ -z "$ONLY" ] || [ "$ONLY" = c5 ]; then
  STEPS=1 run --global-nx 4096
fi
