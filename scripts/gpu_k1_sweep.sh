# K1 sweep: raw headline bench under env settings given as arguments ("BBX_CW_ROWS=32" ...)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --workloads raw --steps 30 --warmup 5 --cpu-seconds 0.5 > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "import json;d=json.load(open('gpurun_out/sweep.json'));r=d['roofline'];print('$cfg', 'value',round(d['value']),'kernel_us',round(r['kernel_us'],1),'frac',round(r['frac'],3))" || tail -3 gpurun_out/sweep.err
done
