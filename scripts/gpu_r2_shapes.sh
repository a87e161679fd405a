#!/bin/bash
# Bench-shape parity tests + a JPEG-only bench leg (round-2 first GPU check).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/shapes.log 2>&1
echo "shapes rc=$?" >> gpurun_out/shapes.log
timeout 600 python bench.py --workloads jpeg --steps 30 --warmup 5 > gpurun_out/bench_jpeg.json 2> gpurun_out/bench_jpeg.err
echo "bench rc=$?"
tail -3 gpurun_out/shapes.log
