#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over scripts/sanitize_driver.py variants.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sanitize
for v in ${VARIANTS:-tma tma3 notmem cpasync noks fuse face fields profiles}; do
  timeout 300 python scripts/sanitize_driver.py $v > gpurun_out/sanitize/plain_$v.log 2>&1 || { echo "plain $v failed" >> gpurun_out/sanitize/summary.txt; continue; }
  for tool in ${TOOLS:-memcheck racecheck synccheck}; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_driver.py $v \
      > gpurun_out/sanitize/${tool}_$v.log 2>&1
    echo "$tool $v exit $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_driver' gpurun_out/sanitize/${tool}_$v.log | tr '\n' ' ')" >> gpurun_out/sanitize/summary.txt
  done
done
