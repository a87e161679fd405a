# One GPU round trip: build, smoke, GPU tests, bench, ncu launch list + full capture of K1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
if [ "${TESTS:-1}" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q --tb=short ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps ${STEPS:-50} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for v in ${VARIANTS:-}; do
  env $v timeout 600 python bench.py --steps ${STEPS:-50} --warmup 5 --cpu-seconds 1 > gpurun_out/bench_$v.json 2>/dev/null; echo "variant $v:"; python -c "import json;d=json.load(open('gpurun_out/bench_$v.json'));print(d['value'], d['e2e'])"
done
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_kernel -s 4 -c 2 -o gpurun_out/prof_k1 -f python bench.py --steps 4 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
fi
