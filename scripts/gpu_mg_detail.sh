#!/bin/bash
# Per-level MG kernel times (TPMG_PROF_DETAIL=1, stderr at destroy) at N = 1 and N = 2,
# exchanges off (timing only) and on, to attribute the N > 1 overhead per kernel and level.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-mgd}
N=$(nvidia-smi -L | wc -l)
export TPMG_PROF_DETAIL=1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --solver mg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/det_${TAG}_n1.json 2> gpurun_out/det_${TAG}_n1.err
i=1
for v in "TPMG_HALO=off" "TPMG_HALO=off TPMG_KSPLIT=0" "TPMG_OVERLAP=0" ""; do
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
    --master-port $((29850 + i)) bench.py --gpus $N --solver mg --steps 3 --warmup 3 --no-e2e \
    > gpurun_out/det_${TAG}_v$i.json 2> gpurun_out/det_${TAG}_v$i.err
  echo "variant $i ($v) exit $?" >> gpurun_out/det_${TAG}.log
  i=$((i + 1))
done
