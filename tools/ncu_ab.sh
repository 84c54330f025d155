for lib in "$@"; do
  HPS_LIBRARY=$PWD/paper_2111_10635_b200/$lib ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ncu_ab_$lib.csv python tools/sweep_once.py --count 4194304 --repeat 1 > /dev/null 2>&1
done
