"""Time the pieces of an epoch iterator's start (pipeline fill) on the raw leg."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12517_b200 as bx  # noqa: E402

path = bench.ensure_dataset(0, lambda: None)
ds, ld = bench.make_loader(path, 0, 0, 1, bx.DeviceResident(0), slot_count=6)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it = ld.iterate_steps(40, start_epoch=rep)
    t1 = time.perf_counter()
    b = next(it)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(39):
        b = next(it)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    it.close()
    print(f"create {1e3*(t1-t0):.3f} ms  first batch {1e3*(t2-t1):.3f} ms  next 39: {1e3*(t3-t2)/39:.3f} ms/step")
