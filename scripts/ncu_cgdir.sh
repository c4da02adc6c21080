cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_1402_3545_b200.build > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_write.sum
for s in "1024 1024" "4096 1024" "4096 4096"; do
  timeout 300 python scripts/cgdir_probe.py $s > /dev/null 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_line" --csv python scripts/cgdir_probe.py $s > gpurun_out/ncu_cgdir_${s// /x}.csv 2>&1
done
