#!/bin/bash
# Bench the headline leg with each variants/libbbx_*.so in place of libbbx.so.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2306_12517_b200/libbbx.so /tmp/libbbx_orig.so
for v in variants/libbbx_*.so; do
  n=$(basename $v .so); cp $v paper_2306_12517_b200/libbbx.so
  for i in 1 2; do
    timeout 300 python bench.py --workloads ${WL:-raw} --steps 30 --warmup 5 --cpu-seconds 0.2 > gpurun_out/var_$n.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/var_$n.json'));r=d['roofline'];print('$n','value',round(d['value']),'kernel_us',round(r['kernel_us'],1),'frac',round(r['frac'],3))"
  done
  if [ -n "$NCU" ]; then
    timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,launch__shared_mem_per_block_dynamic --clock-control none -k regex:image_cw_kernel -s 4 -c 3 python bench.py --workloads raw --steps 3 --warmup 3 --cpu-seconds 0.2 2>/dev/null | grep -E "duration|inst_executed|dram|occupancy|warps_active|shared_mem" | tail -7
  fi
done
cp /tmp/libbbx_orig.so paper_2306_12517_b200/libbbx.so
