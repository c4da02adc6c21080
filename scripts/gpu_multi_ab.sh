#!/bin/bash
# Multi-GPU A/B: parity tests, then N-rank bench with P2P halos vs NCCL halos.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r1}
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/mr_pytest_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/mr_pytest_$TAG.log
i=0
for halo in ${HALOS:-p2p nccl p2p nccl}; do
  i=$((i+1))
  TPMG_HALO=$halo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + i)) bench.py --gpus $N --steps 4 --warmup 3 --no-e2e > gpurun_out/bench_n${N}_${halo}${i}_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/bench_n${N}_${halo}${i}_$TAG.log
done
