# Bench both workloads, then the ncu launch list and one full capture of a named kernel.
# env: STEPS (30), KERNEL (regex for the full capture, default jpeg_huffman_kernel), WL (jpeg)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-30} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${WL:-jpeg}.csv python bench.py --workloads ${WL:-jpeg} --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-jpeg_huffman_kernel} -s 4 -c 1 -o gpurun_out/prof_full -f python bench.py --workloads ${WL:-jpeg} --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
fi
