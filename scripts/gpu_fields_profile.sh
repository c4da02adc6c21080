#!/bin/bash
# GPU box: full checks of the current build plus a full ncu capture of the per-column-fields
# line kernels (smoother, preconditioner, residual) at 1024^2 x 128.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r1v}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
PROF_FIELDS=smooth timeout 300 python scripts/profile_kernels.py > gpurun_out/prof_fields_plain_$TAG.log 2>&1 && \
PROF_FIELDS=smooth timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_line" -c 3 \
    -o gpurun_out/proff_$TAG python scripts/profile_kernels.py > gpurun_out/ncu_fields_$TAG.log 2>&1
echo "fields capture exit $?" >> gpurun_out/ncu_fields_$TAG.log
if [ -f gpurun_out/proff_$TAG.ncu-rep ]; then
  ncu -i gpurun_out/proff_$TAG.ncu-rep --page raw --csv > gpurun_out/proff_${TAG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/proff_$TAG.ncu-rep --page details --csv > gpurun_out/proff_${TAG}_details.csv 2>/dev/null
  rm -f gpurun_out/proff_$TAG.ncu-rep
fi
