cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_1402_3545_b200.build > /dev/null 2>&1
for cfg in ${CFGS:-"2048 4" "16384 4" "16384 8" "4096 4" "65536 2" "262144 1"}; do
  set -- $cfg
  TPMG_PROLONG_WANT=$1 TPMG_PROLONG_MINLPT=$2 timeout 120 python scripts/prolong_ab.py 2>&1 | tail -1
done > gpurun_out/prolong_ab.txt
