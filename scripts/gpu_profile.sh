#!/bin/bash
# GPU-box profiling pass (run under gpurun from the repo root): launch list of the
# bench command and one full ncu capture of the hot kernels.  Each ncu run follows a
# plain run of the same command that exited 0.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
BENCH="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $BENCH > gpurun_out/bench_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $BENCH > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_$TAG.log
timeout 300 python scripts/profile_kernels.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k_line" -c ${NCU_COUNT:-12} \
    -o gpurun_out/prof_$TAG python scripts/profile_kernels.py > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture exit $?" >> gpurun_out/ncu_full_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_prolong" -c 4 \
    -o gpurun_out/profp_$TAG python scripts/profile_kernels.py > gpurun_out/ncu_fullp_$TAG.log 2>&1
echo "prolong capture exit $?" >> gpurun_out/ncu_fullp_$TAG.log
# raw metric exports travel back; reports only when small (gpurun copies <= 64 MiB)
for r in prof profp; do
  [ -f gpurun_out/${r}_$TAG.ncu-rep ] || continue
  ncu -i gpurun_out/${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/${r}_${TAG}_raw.csv 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/${r}_$TAG.ncu-rep
done
