#!/bin/bash
# Multi-GPU pass (gpurun --gpus N): multirank parity tests, then bench A/B at N ranks:
# default (P2P halos overlapped, NVLink allreduce) vs TPMG_OVERLAP=0 vs TPMG_ALLREDUCE=nccl
# vs TPMG_HALO=nccl.  Per-rank MG / PCG times from the JSON line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-mr}
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_$TAG.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest ${PYTEST_FILES:-tests/test_gpu_multirank.py tests/test_gpu_halo.py} -m gpu -q -rs > gpurun_out/pytest_multirank_${N}gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_multirank_${N}gpu_$TAG.log
fi
IFS=';' read -ra VS <<< "${VARIANTS:--;TPMG_OVERLAP=0;TPMG_ALLREDUCE=nccl;TPMG_HALO=nccl}"
for rep in $(seq 1 ${REPS:-2}); do
  for i in "${!VS[@]}"; do
    v="${VS[$i]}"; [ "$v" = "-" ] && v=""
    env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
      --master-port $((29700 + i + 10 * rep)) bench.py --gpus $N --steps ${STEPS:-5} --warmup 3 --no-e2e ${BENCH_ARGS} \
      > gpurun_out/ab_${TAG}_${i}_${rep}.json 2> gpurun_out/ab_${TAG}_${i}_${rep}.err
    echo "variant $i ($v) rep $rep exit $?" >> gpurun_out/ab_${TAG}.log
  done
done
