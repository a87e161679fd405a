# Round evidence: GPU tests, smoke, full bench line, launch lists (raw, jpeg), ncu full capture of K1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final_launches_raw.csv python bench.py --workloads raw --steps 4 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu_raw rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/final_launches_jpeg.csv python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu_jpeg rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:image_cw_kernel -s 4 -c 1 -o gpurun_out/final_k1 -f python bench.py --workloads raw --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/final_ncu_k1.log 2>&1; echo ncu_k1 rc=$?
