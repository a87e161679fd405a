# JPEG iteration: GPU JPEG tests, then a launch list of the configs[2] leg
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jpeg.py -x -q > gpurun_out/pytest_jpeg.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_jpeg.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_jq.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu rc=$?
python scripts/launch_summary.py gpurun_out/launches_jq.csv
