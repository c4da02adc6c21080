#!/bin/bash
# Multi-GPU pass (run under gpurun --gpus N): multi-rank parity tests, then the bench at N.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r1}
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/mr_pytest_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/mr_pytest_$TAG.log
for n in $(seq 2 $N); do
  case $n in 2|4|8) ;; *) continue;; esac
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n ${BENCH_ARGS:---steps 3 --warmup 2} > gpurun_out/bench_n${n}_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/bench_n${n}_$TAG.log
done
