#!/bin/bash
# MG multi-GPU overhead probe (gpurun --gpus 2): the same per-GPU workload (1024^2 x 128,
# MG only) at N = 1 and N = 2 on one box, N = 2 with the halo exchanges on / off
# (TPMG_HALO=off: timing only, wrong results), overlap on / off, NVLink / NCCL allreduce.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-mgo}
N=$(nvidia-smi -L | wc -l)
for rep in 1 2; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --solver mg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_0_${rep}.json 2> gpurun_out/ab_${TAG}_0_${rep}.err
  i=1
  for v in "" "TPMG_OVERLAP=0" "TPMG_HALO=off" "TPMG_HALO=off TPMG_ALLREDUCE=nccl" "TPMG_HALO=nccl"; do
    env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
      --master-port $((29800 + i + 10 * rep)) bench.py --gpus $N --solver mg --steps 10 --warmup 3 --no-e2e \
      > gpurun_out/ab_${TAG}_${i}_${rep}.json 2> gpurun_out/ab_${TAG}_${i}_${rep}.err
    echo "variant $i ($v) rep $rep exit $?" >> gpurun_out/ab_${TAG}.log
    i=$((i + 1))
  done
done
