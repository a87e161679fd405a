"""K1 time per launch vs batch size at the configs[1] chain (HBM-resident heap, one
compute stream, every launch timed): separates the per-launch fixed cost (ramp and tail
of the persistent grid) from the per-image cost.  Run on the GPU box."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2306_12517_b200 as bx  # noqa: E402

noop = lambda: None  # noqa: E731
path = bench.raw_dataset(0, noop)
for batch in (128, 256, 512, 1024, 2048):
    ds, ld = bench.make_loader(path, 0, 0, 1, bx.DeviceResident(0), bench.CHAIN_SPEC, "random", batch, 6,
                               options={"compute_streams": 1})
    ld.set_profiling(1)
    it = ld.iterate_steps(60)
    for _ in range(10):
        next(it)
    ld.reset_stats()
    for _ in range(50):
        next(it)
    it.close()
    st = ld.stats()
    us = st["kernel_seconds"] / max(st["kernel_timed"], 1) * 1e6
    print(f"batch {batch:5d}: K1 {us:7.1f} us per launch, {us / batch * 1e3:6.1f} ns per image")
    ld.shutdown()
    ds.close()
