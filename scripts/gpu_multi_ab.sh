#!/bin/bash
# Multi-GPU A/B: parity tests, then N-rank bench with overlap on / off.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r1}
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/mr_pytest_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/mr_pytest_$TAG.log
for ov in 1 0; do
  TPMG_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + ov)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e > gpurun_out/bench_n${N}_ov${ov}_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/bench_n${N}_ov${ov}_$TAG.log
done
