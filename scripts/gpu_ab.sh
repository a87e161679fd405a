# A/B of variants/libbbx_*.so on one bench leg, interleaved rounds: WL=<workloads> KEY=<leg> bash scripts/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2306_12517_b200/libbbx.so /tmp/libbbx_orig.so
for round in 1 2 3; do
  for v in variants/libbbx_*.so; do
    n=$(basename $v .so); cp $v paper_2306_12517_b200/libbbx.so
    timeout 300 python bench.py --details gpurun_out/_details.json --workloads ${WL:-jpeg} --steps ${STEPS:-30} --warmup 5 --cpu-seconds 0.2 > gpurun_out/ab_$n.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/_details.json'))
w=d['workloads']['${KEY:-configs[2]}']; print('$n', round(w['value']), 'ms', round(w['ms_per_step'],4), 'dev', round(w.get('device_ms_per_batch',0),4), 'e2e', round(w['e2e']['value']), w.get('parity_ok'))"
  done
done
cp /tmp/libbbx_orig.so paper_2306_12517_b200/libbbx.so
if [ -n "$NCU" ]; then
  for v in variants/libbbx_*.so; do
    n=$(basename $v .so); cp $v paper_2306_12517_b200/libbbx.so
    echo $n; timeout 300 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:${NCU_K:-huffman} -s 2 -c 1 python bench.py --details gpurun_out/_details.json --workloads ${WL:-jpeg} --steps 3 --warmup 3 --cpu-seconds 0.2 2>/dev/null | grep -E "duration|occupancy|warps_active"
  done
  cp /tmp/libbbx_orig.so paper_2306_12517_b200/libbbx.so
fi
