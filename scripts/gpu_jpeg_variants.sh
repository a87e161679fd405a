# JPEG A/B: GPU JPEG parity tests with each variants/libbbx_*.so, then interleaved configs[2] benches and J2 ncu times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2306_12517_b200/libbbx.so /tmp/libbbx_orig.so
for v in variants/libbbx_*.so; do
  n=$(basename $v .so); cp $v paper_2306_12517_b200/libbbx.so
  timeout 900 python -m pytest tests/test_gpu_jpeg.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/jv_pytest_$n.log 2>&1; echo $n pytest rc=$?; tail -1 gpurun_out/jv_pytest_$n.log
  echo $n; timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:${NCU_K:-huffman} -s 4 -c 2 python bench.py --workloads jpeg --steps 3 --warmup 3 --cpu-seconds 0.2 2>/dev/null | grep -E "duration|inst_exec"
done
cp /tmp/libbbx_orig.so paper_2306_12517_b200/libbbx.so
bash scripts/gpu_ab.sh
