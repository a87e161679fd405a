"""Page-cache golden counts from the UNMODIFIED reference (reader.py:96-145
PageSchedule, loader.py:273-291,443-445 EpochStats):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_page_golden.py

Writes tests/golden/page_cases.json:
  traces:  [trace, capacity, planned_fetches, planned_reloads] -- the example and
           random traces of tests/test_reader_cache.py:106-127 (rng 17)
  loader:  reference Loader epochs over the committed paged.bbox fixture with a
           ProcessCacheStrategy: batch indices + EpochStats page_fetches/reloads
"""

import json
from pathlib import Path

import numpy as np

from bbox import LoaderConfig, Loader, OrderKind, ProcessCacheStrategy, open_dataset
from bbox.errors import CapacityTooSmall
from bbox.reader import PageSchedule

HERE = Path(__file__).resolve().parent


def main():
    traces = []
    ex = [0, 1, 2, 3, 4, 5, 0, 1, 2, 3, 4, 5]
    for cap in (1, 2, 3, 4, 6):
        s = PageSchedule(ex, cap)
        traces.append([ex, cap, s.planned_fetches, s.planned_reloads])
    rng = np.random.default_rng(17)
    for _ in range(150):
        pages = int(rng.integers(1, 20))
        trace = [int(p) for p in rng.integers(0, pages, size=int(rng.integers(1, 120)))]
        cap = int(rng.integers(1, 10))
        s = PageSchedule(trace, cap)
        traces.append([trace, cap, s.planned_fetches, s.planned_reloads])
    loader_cases = []
    path = HERE / "paged.bbox"
    for order, cap, bs, seed, epoch in [("quasi-random", 6, 6, 4, 0), ("quasi-random", 3, 8, 2, 1),
                                        ("random", 10, 4, 1, 0), ("random", 4, 2, 7, 2),
                                        ("sequential", 2, 16, 0, 0), ("random", 1, 64, 1, 0), ("quasi-random", 10, 20, 9, 3)]:
        ds = open_dataset(path, ProcessCacheStrategy(capacity_pages=cap, prefetch_window=4))
        try:
            cfg = LoaderConfig(batch_size=bs, num_workers=2, order=OrderKind(order), seed=seed)
            loader = Loader(ds, cfg)
            case = {"order": order, "capacity": cap, "batch_size": bs, "seed": seed, "epoch": epoch,
                    "num_pages": ds.num_pages}
            try:
                case["batches"] = [list(b.indices) for b in loader.iterate_epoch(epoch)]
                case["page_fetches"] = loader.last_stats.page_fetches
                case["page_reloads"] = loader.last_stats.page_reloads
            except CapacityTooSmall as e:
                case["error"] = str(e)
            loader_cases.append(case)
        finally:
            ds.close()
    (HERE / "page_cases.json").write_text(json.dumps({"traces": traces, "loader": loader_cases}))
    print(len(traces), "traces,", len(loader_cases), "loader cases")


if __name__ == "__main__":
    main()
