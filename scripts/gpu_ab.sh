#!/bin/bash
# Generic A/B on one GPU (run under gpurun from the repo root): for each variant in VARIANTS
# (";"-separated lists of env assignments, "-" = defaults), REPS alternations of
#   python bench.py $BENCH_ARGS
# -> gpurun_out/ab_<TAG>_<variant index>_<rep>.json.  Optional pytest -m gpu first (TESTS=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-ab}
REPS=${REPS:-2}
BENCH_ARGS=${BENCH_ARGS:---solver cg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e}
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_SEL} > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
IFS=';' read -ra VS <<< "${VARIANTS:--}"
for rep in $(seq 1 $REPS); do
  for i in "${!VS[@]}"; do
    v="${VS[$i]}"; [ "$v" = "-" ] && v=""
    env $v timeout 600 python bench.py $BENCH_ARGS > gpurun_out/ab_${TAG}_${i}_${rep}.json 2> gpurun_out/ab_${TAG}_${i}_${rep}.err
    echo "variant $i ($v) rep $rep exit $?" >> gpurun_out/ab_${TAG}.log
  done
done
