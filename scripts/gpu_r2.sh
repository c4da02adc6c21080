#!/bin/bash
# Round-2 GPU pass (run under gpurun from the repo root): GPU tests, then an A/B of the
# Thomas g' buffer in Tensor Memory (TPMG_TMEM=1, default) vs shared memory (TPMG_TMEM=0)
# on the CG step, then a short default bench.  TAG names the output files.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_SEL} > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
for rep in 1 2; do
  for tm in 1 0; do
    TPMG_TMEM=$tm timeout 300 python bench.py --solver cg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/ab_tmem${tm}_${rep}_$TAG.json 2>gpurun_out/ab_tmem${tm}_${rep}_$TAG.err
  done
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench exit $?" >> gpurun_out/bench_$TAG.err
