#!/bin/bash
# JPEG iteration: JPEG GPU parity tests, configs[2] bench leg, launch list (per-kernel means).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jpeg.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/pytest_jpeg.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_jpeg.log
timeout 600 python bench.py --workloads jpeg --steps 30 --warmup 5 --cpu-seconds 0.5 > gpurun_out/bench_jpeg.json 2> gpurun_out/bench_jpeg.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_jpeg.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.2 > /dev/null 2>&1; echo ncu rc=$?
python scripts/launch_summary.py gpurun_out/launches_jpeg.csv > gpurun_out/launches_jpeg_summary.txt 2>&1; cat gpurun_out/launches_jpeg_summary.txt
