#!/bin/bash
# ncu --set full of the CG kernels (k_line modes 4 and 5) at 1024^2 x 128, after a plain run
# of the same command exits 0; exports the raw page and the source page of the iteration's
# CGPREC (the third captured launch).  Extra env (e.g. TPMG_TM_CTAS) passes through.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r2b}
timeout 300 python scripts/profile_kernels.py > gpurun_out/prof_plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    ${NCU_EXTRA} -k regex:"k_line<.int.[45]," -c ${NCU_COUNT:-3} -o gpurun_out/cg_$TAG python scripts/profile_kernels.py \
    > gpurun_out/ncu_cg_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_cg_$TAG.log
ncu -i gpurun_out/cg_$TAG.ncu-rep --page raw --csv > gpurun_out/cg_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/cg_$TAG.ncu-rep --page source --csv --kernel-name-base demangled -k regex:"k_line<.int.5," \
    --launch-skip 1 --launch-count 1 > gpurun_out/cg_${TAG}_source.csv 2>/dev/null
ls -la gpurun_out/cg_$TAG.ncu-rep >> gpurun_out/ncu_cg_$TAG.log
