#!/bin/bash
# Multi-rank timing probe: per-V-cycle and per-CG-iteration time (max over ranks) for the
# halo variants, at N = 1, 2 and all GPUs of the box.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_1402_3545_b200.build > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
i=0
for n in 1 2 $N; do
  for h in ${VARIANTS:-p2p p2p-fused nccl off}; do
    i=$((i+1))
    [ $n -eq 1 ] && [ $h != p2p ] && continue
    fp=0; hh=$h
    [ $h = p2p-fused ] && fp=1 && hh=p2p
    TPMG_HALO=$hh TPMG_FUSED_PUSH=$fp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29800 + i)) scripts/mr_probe.py 2>&1 | grep "^N=" | sed "s/\$/ fused_push=$fp/"
  done
done > gpurun_out/mr_probe.txt
