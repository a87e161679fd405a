#!/bin/bash
# Host topology facts for DESIGN §6 (NUMA node of the GPU, cores, memory bandwidth).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ lscpu | head -30; echo; nvidia-smi topo -m; echo; for n in /sys/devices/system/node/node*; do echo $n $(cat $n/cpulist); done;
  bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^00000000/0000/');
  echo gpu $bus numa_node $(cat /sys/bus/pci/devices/$bus/numa_node 2>/dev/null); free -g; } > gpurun_out/topo.txt 2>&1
python - <<'PY' >> gpurun_out/topo.txt 2>&1
import numpy as np, time, threading, os
# host memcpy bandwidth: 1 and N threads, 256 MB buffers each
def bw(nt):
    srcs=[np.ones(64<<20, np.uint32) for _ in range(nt)]; dsts=[np.empty_like(s) for s in srcs]
    for s,d in zip(srcs,dsts): np.copyto(d,s)
    t0=time.perf_counter()
    ths=[threading.Thread(target=lambda s=s,d=d: [np.copyto(d,s) for _ in range(4)]) for s,d in zip(srcs,dsts)]
    [t.start() for t in ths]; [t.join() for t in ths]
    el=time.perf_counter()-t0
    return nt*4*(256<<20)*2/el/1e9
for nt in (1, 4, 8, 16, os.cpu_count()):
    print("memcpy threads", nt, "GB/s (read+write)", round(bw(nt),1))
PY
cat gpurun_out/topo.txt | tail -25
