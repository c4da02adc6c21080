#!/bin/bash
# Scaling pass on an N-GPU box (gpurun --gpus N): multi-rank parity, then
#   weak scaling at 1024^2 x 128 per GPU (the bench default) and 2048^2 x 128 per GPU (C4),
#   strong scaling of 4096^2 x 128 (C5), each at N = 1, 2, 4 (as many as the box has).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r1}
python -m paper_1402_3545_b200.build > /dev/null 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/mr_pytest_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/mr_pytest_$TAG.log
fi
run() {   # run <n> <tag> <bench args...>
  local n=$1 t=$2; shift 2
  if [ $n -eq 1 ]; then
    timeout 900 python bench.py "$@" > gpurun_out/scale_${TAG}_${t}_n1.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29650 + n)) bench.py --gpus $n "$@" > gpurun_out/scale_${TAG}_${t}_n$n.log 2>&1
  fi
  echo "exit $?" >> gpurun_out/scale_${TAG}_${t}_n$n.log
}
for n in 1 2 4; do
  [ $n -le $N ] || continue
  run $n weak1024 --steps 3 --warmup 3 --no-cpu-baseline
  run $n weak2048 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --per-gpu-nx 2048
  run $n strong4096 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --global-nx 4096
done
