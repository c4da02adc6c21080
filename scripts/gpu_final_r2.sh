#!/bin/bash
# Final single-GPU evidence of the round (run under gpurun from the repo root):
#   build + smoke, the GPU test suite, the driver's bench command (both arms), the launch list
#   of a bench step (ncu gpu__time_duration, after the plain run exits 0), and one ncu --set full
#   capture of the line kernels and the prolongation (profile_kernels.py), exported as CSV.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
t0=$SECONDS; timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "wall $((SECONDS - t0)) s" >> gpurun_out/bench_ref_$TAG.err
t0=$SECONDS; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "wall $((SECONDS - t0)) s" >> gpurun_out/bench_$TAG.err
[ -n "$SKIP_NCU" ] && exit 0
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $BENCH > gpurun_out/bench_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $BENCH > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_$TAG.log
timeout 300 python scripts/profile_kernels.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_line|k_prolong" -c ${NCU_COUNT:-40} -o gpurun_out/prof_$TAG python scripts/profile_kernels.py \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture exit $?" >> gpurun_out/ncu_full_$TAG.log
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --kernel-name-base demangled -k regex:"k_line<.int.5," \
    --launch-skip 1 --launch-count 1 > gpurun_out/prof_${TAG}_cgprec_source.csv 2>/dev/null
[ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_$TAG.ncu-rep
