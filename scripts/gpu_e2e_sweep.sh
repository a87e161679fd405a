# e2e sweep over staging threads
cd $GRAFT_REPO_ROOT
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node" | head -8
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --workloads raw --steps 30 --warmup 5 --cpu-seconds 0.5 > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "import json;d=json.load(open('gpurun_out/sweep.json'));e=d['e2e'];z=d['e2e_zero_copy'];print('$cfg', 'e2e',round(e['value']),'stage_ms',round(e['host_stage_ms_per_step'],3),'gbs',round(e['h2d_gbs'],1),'zc',round(z['value']))" || tail -3 gpurun_out/sweep.err
done
