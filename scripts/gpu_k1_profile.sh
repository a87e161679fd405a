# K1 evidence: raw launch list + one ncu --set full capture of image_cw_kernel + bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_raw.csv python bench.py --workloads raw --steps 4 --warmup 3 --cpu-seconds 0.5 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:image_cw_kernel -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --workloads raw --steps 3 --warmup 3 --cpu-seconds 0.5 > gpurun_out/ncu_k1.log 2>&1; echo ncu2 rc=$?
