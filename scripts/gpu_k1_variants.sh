# K1 A/B: bench-shape parity tests with each variants/libbbx_*.so, then the variant benches (gpu_variants.sh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2306_12517_b200/libbbx.so /tmp/libbbx_orig.so
for v in variants/libbbx_*.so; do
  n=$(basename $v .so); cp $v paper_2306_12517_b200/libbbx.so
  timeout 900 python -m pytest tests/test_gpu_k1.py tests/test_gpu_bench_shapes.py -x -q -m gpu > gpurun_out/k1_pytest_$n.log 2>&1; echo $n pytest rc=$?; tail -1 gpurun_out/k1_pytest_$n.log
done
cp /tmp/libbbx_orig.so paper_2306_12517_b200/libbbx.so
NCU=1 bash scripts/gpu_variants.sh
