#!/bin/bash
# Wide grids: PCG kernel bandwidth vs nx (powers of two and not), tile bands, and ncu of the
# CG kernels at 4096^2 (DRAM bytes vs algorithmic, L2 hit rate).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-wide}
for cfg in "1024" "2048" "2000" "4096" "4000" "4096 TPMG_BAND=32" "4096 TPMG_BAND=8"; do
  set -- $cfg
  nx=$1; shift
  name=$(echo "$nx $*" | sed 's/[ =]//g')
  env "$@" timeout 900 python bench.py --global-nx $nx --solver cg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/wide_${TAG}_${name}.json 2> gpurun_out/wide_${TAG}_${name}.err
done
for n in ${NCU_SIZES:-4096 4000}; do
  PROF_N=$n PROF_CG_ONLY=1 timeout 300 python scripts/profile_kernels.py > gpurun_out/prof_wide_${TAG}_$n.log 2>&1 || continue
  PROF_N=$n PROF_CG_ONLY=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"k_line<.int.[45]," -c 3 -o gpurun_out/wide_${TAG}_$n python scripts/profile_kernels.py \
      > gpurun_out/ncu_wide_${TAG}_$n.log 2>&1
  ncu -i gpurun_out/wide_${TAG}_$n.ncu-rep --page raw --csv > gpurun_out/wide_${TAG}_${n}_raw.csv 2>/dev/null
  rm -f gpurun_out/wide_${TAG}_$n.ncu-rep   # (the pull-back limit is 64 MiB)
done
