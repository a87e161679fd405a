# JPEG iteration: GPU JPEG parity tests, the configs[2] bench leg (twice), and its launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jpeg.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/jq_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/jq_pytest.log
for i in 1 2; do timeout 600 python bench.py --details gpurun_out/_details.json --workloads jpeg --steps 30 --warmup 5 --cpu-seconds 0.3 > gpurun_out/jq_bench.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/_details.json'))
for k,w in d['workloads'].items(): print(k, round(w['value']), 'ms', round(w['ms_per_step'],4), 'dev', round(w.get('device_ms_per_batch',0),4), 'prep', round(w.get('host_prep_ms_per_step',0),4), 'e2e', round(w['e2e']['value']), w.get('parity_ok'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:jpeg_huffman -c 6 --csv --log-file gpurun_out/jq_launches.csv python bench.py --details gpurun_out/_details.json --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/jq_launches.csv')))
hi=next(i for i,r in enumerate(rows) if 'Metric Name' in r); h=rows[hi]
for r in rows[hi+1:]:
    if len(r)>h.index('Metric Value'): print(r[h.index('Metric Name')], r[h.index('Metric Value')])
PY
