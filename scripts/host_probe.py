"""Host-side cost per step of the HBM-resident legs (configs[0], configs[1]): step time,
the consumer's time inside next(), and the pipeline thread's descriptor time, for a few
values of the loader option parallel_desc_min.  Run on the GPU box."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_12517_b200 as bx  # noqa: E402

noop = lambda: None  # noqa: E731
for leg, path, chain in (("configs[0]", bench.cifar_dataset(0, noop), bench.CIFAR_SPEC),
                         ("configs[1]", bench.raw_dataset(0, noop), bench.CHAIN_SPEC)):
    for pmin in (256, 1 << 30):
        ds, ld = bench.make_loader(path, 0, 0, 1, bx.DeviceResident(0), chain, "random", bench.B, 6,
                                   options={"parallel_desc_min": pmin})
        it = ld.iterate_steps(400)
        for _ in range(50):
            next(it)
        torch.cuda.synchronize()
        ld.reset_stats()
        t_next = 0.0
        t0 = time.perf_counter()
        for _ in range(300):
            a = time.perf_counter()
            b = next(it)
            t_next += time.perf_counter() - a
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        st = ld.stats()
        print(f"{leg} parallel_desc_min={pmin}: step {el / 300 * 1e6:.1f} us, consumer in next() {t_next / 300 * 1e6:.1f} us, "
              f"pipeline {st['pipeline_seconds'] / max(st['batches'], 1) * 1e6:.1f} us (desc/stage {st['stage_seconds'] / max(st['batches'], 1) * 1e6:.1f}), wait {st['wait_seconds'] / 300 * 1e6:.1f} us")
        it.close()
        ld.shutdown()
        ds.close()
