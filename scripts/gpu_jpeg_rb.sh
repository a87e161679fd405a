# J2 time per restart interval setting (launch list per setting)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rb in ${RBS:-4 2 1}; do
  BBX_BENCH_RST_BLOCKS=$rb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_rb$rb.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.2 > /dev/null 2>&1
  echo "rst_blocks=$rb"; python scripts/launch_summary.py gpurun_out/launches_rb$rb.csv | head -6
done
