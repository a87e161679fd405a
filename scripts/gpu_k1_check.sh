#!/bin/bash
# K1 iteration: all GPU tests, then the headline (raw) bench leg twice, then an ncu capture of K1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_k1.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_k1.log
for i in 1 2; do
timeout 600 python bench.py --workloads raw --steps 30 --warmup 5 --cpu-seconds 0.5 > gpurun_out/bench_k1_$i.json 2> gpurun_out/bench_k1_$i.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_k1_$i.json'));r=d['roofline'];print('value',round(d['value']),'kernel_us',round(r['kernel_us'],1),'frac',round(r['frac'],3),'e2e',round(d['e2e']['value']))"
done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:image_cw_kernel -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --workloads raw --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/ncu_k1.log 2>&1; echo ncu rc=$?
fi
