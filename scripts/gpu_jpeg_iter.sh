# JPEG iteration: parity tests, bench per restart interval, launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_jpeg.py -q -x --tb=short 2>&1 | tail -15
for rb in ${RBS:-4}; do
  BBX_BENCH_RST_BLOCKS=$rb timeout 300 python bench.py --workloads jpeg --steps 30 --warmup 5 --cpu-seconds 1 2>gpurun_out/bench_rb$rb.err | tail -1 > gpurun_out/bench_rb$rb.json
  python -c "import json; d=json.load(open('gpurun_out/bench_rb$rb.json')); j=d['workloads']['configs[2]']; print('rst_blocks=$rb', 'value', round(j['value']), 'dev_ms', round(j['device_ms_per_batch'],3), 'e2e', round(j['e2e']['value']), 'stage_ms', round(j['e2e']['host_stage_ms_per_step'],3), 'h2d/img', round(j['h2d_bytes_per_image']))" || tail -5 gpurun_out/bench_rb$rb.err
done
BBX_BENCH_RST_BLOCKS=${RBS%% *} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_jpeg3.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.2 > /dev/null 2>&1; echo ncu rc=$?
python scripts/launch_summary.py gpurun_out/launches_jpeg3.csv
