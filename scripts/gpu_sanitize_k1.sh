# compute-sanitizer memcheck / racecheck / synccheck on K1 (image_cw_kernel) over the small RRC parity cases
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=image_cw_kernel python -m pytest tests/test_gpu_k1.py -x -q -m gpu -k "${SAN_K:-rrc}" > gpurun_out/${T}_san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/${T}_san_$tool.log | tail -3
done
