#!/bin/bash
# 4-GPU pass: multirank parity (all cases), then weak scaling at 1024^2 and 2048^2 per GPU
# and strong scaling of 4096^2 (C5) at N = 1, 2, 4 (default build and options).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-sc}
N=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_halo.py -m gpu -q -rs > gpurun_out/pytest_multirank_${N}gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_multirank_${N}gpu_$TAG.log
for cfg in "--per-gpu-nx 1024" "--per-gpu-nx 2048" "--global-nx 4096"; do
  name=$(echo $cfg | tr -d ' -')
  for n in 1 2 4; do
    [ $n -gt $N ] && continue
    if [ $n -eq 1 ]; then
      timeout 900 python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/scale_${TAG}_${name}_n1.json 2> gpurun_out/scale_${TAG}_${name}_n1.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port $((29900 + n)) \
        bench.py --gpus $n $cfg --steps 5 --warmup 3 --no-e2e > gpurun_out/scale_${TAG}_${name}_n$n.json 2> gpurun_out/scale_${TAG}_${name}_n$n.err
    fi
    echo "$cfg n=$n exit $?" >> gpurun_out/scale_${TAG}.log
  done
done
