cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/q_pytest.log
for i in 1 2; do timeout 600 python bench.py --details gpurun_out/_details.json --workloads raw,cifar --steps 100 --warmup 5 --cpu-seconds 0.3 > gpurun_out/q_bench.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/_details.json'))
for k,w in d['workloads'].items(): print(k, round(w['value']), 'ms', round(w['ms_per_step'],4), 'dev', round(w.get('device_ms_per_batch',0),4), 'prep', round(w.get('host_prep_ms_per_step',0),4), 'e2e', round(w['e2e']['value']))"
done
