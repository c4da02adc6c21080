#!/bin/bash
# Default bench exactly as the driver runs it (N=1, no flags), plus clocks, then profiling.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/bench_default_$TAG.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/bench_reference_$TAG.log
nproc > gpurun_out/host_$TAG.txt; lscpu | head -20 >> gpurun_out/host_$TAG.txt; free -g >> gpurun_out/host_$TAG.txt
