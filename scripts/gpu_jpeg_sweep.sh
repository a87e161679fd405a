# JPEG launch-list sweep over env settings ("BBX_J2_PER_LANE=2" ...): per-kernel means
cd $GRAFT_REPO_ROOT
for cfg in "$@"; do
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_sw.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1
  echo "== $cfg"; python scripts/launch_summary.py gpurun_out/launches_sw.csv | head -3
done
