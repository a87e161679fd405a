#!/bin/bash
# Round evidence: GPU tests, smoke, default bench line, launch lists (raw, jpeg),
# ncu --set full of K1 (configs[1]) and of the JPEG kernels (configs[2]).
#   scripts/gpu_evidence.sh <tag>
cd "$(dirname "$0")/.."
T=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py --details gpurun_out/${T}_bench_details.json > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches_raw.csv python bench.py --workloads raw --steps 4 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu_raw rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_jpeg.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu_jpeg rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:image_cw_kernel -s 4 -c 1 -o gpurun_out/${T}_k1 -f python bench.py --workloads raw --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/${T}_ncu_k1.log 2>&1; echo ncu_k1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jpeg_ -s 6 -c 3 -o gpurun_out/${T}_jpeg -f python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/${T}_ncu_jpeg.log 2>&1; echo ncu_jpeg_full rc=$?
