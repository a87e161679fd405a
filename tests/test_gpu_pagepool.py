"""HBM page pool (ProcessCacheStrategy, reader.py:96-297): the device pool
executes the reference's Belady PageSchedule batch by batch.  Counts are
checked against the UNMODIFIED reference (tests/golden/page_cases.json,
make_page_golden.py): the traces of tests/test_reader_cache.py:106-127 and
reference Loader epochs over the paged fixture (tests/test_loader.py:122-146),
and every batch read from the pool is bit-exact against the oracle."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O
from paper_2306_12517_b200.errors import CapacityTooSmall

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).parent / "golden"
CASES = json.loads((GOLDEN / "page_cases.json").read_text())


@pytest.fixture(scope="module")
def one_per_page(tmp_path_factory):
    """20 RAW images of 36,000 B at 64 KiB pages: sample j lives alone in page j."""
    path = tmp_path_factory.mktemp("pp") / "one_per_page.bbox"
    bx.write_dataset(bx.SyntheticImageSource(20, 120, 100, 3, seed=5), path, bx.WriterConfig(seed=1, page_size=65536))
    ds = bx.open_dataset(path)
    assert [ds.primary_page(i) for i in range(20)] == list(range(20))
    ds.close()
    return path


def _run_trace(path, trace, capacity):
    ds = bx.open_dataset(path, bx.ProcessCacheStrategy(capacity_pages=capacity))
    cfg = bx.LoaderConfig(batch_size=1, order=bx.OrderKind.SEQUENTIAL, seed=0)
    loader = bx.Loader(ds, cfg)
    loader._epoch_batch_arrays = lambda epoch: [np.array([p], dtype=np.int64) for p in trace]
    got = [(b.indices[0], b["image"].cpu().numpy()[0]) for b in loader.iterate_epoch(0)]
    st = loader.last_stats
    loader.shutdown()
    ds.close()
    return got, st


def test_trace_counts_equal_reference_schedule(one_per_page):
    f = O.OracleFile(one_per_page)
    want_img = {i: O.run_field_batch(f, f.fields[0], 0, O.parse_spec("decode"), [i], 0, 0)[0] for i in range(20)}
    for trace, cap, fetches, reloads in CASES["traces"]:
        got, st = _run_trace(one_per_page, trace, cap)
        assert [g[0] for g in got] == trace
        assert (st.page_fetches, st.page_reloads) == (fetches, reloads), (trace, cap)
        for i, img in got:   # every batch read the right pool slot
            assert np.array_equal(img, want_img[i])


@pytest.mark.parametrize("case", range(len(CASES["loader"])))
def test_loader_epochs_match_reference(case):
    c = CASES["loader"][case]
    path = GOLDEN / "paged.bbox"
    ds = bx.open_dataset(path, bx.ProcessCacheStrategy(capacity_pages=c["capacity"], prefetch_window=4))
    cfg = bx.LoaderConfig(batch_size=c["batch_size"], order=bx.OrderKind(c["order"]), seed=c["seed"])
    with bx.Loader(ds, cfg) as loader:
        if "error" in c:
            with pytest.raises(CapacityTooSmall, match=c["error"]):
                next(iter(loader.iterate_epoch(c["epoch"])))
        else:
            got = [(list(b.indices), b["image"].cpu().numpy(), b["label"].cpu().numpy())
                   for b in loader.iterate_epoch(c["epoch"])]
            st = loader.last_stats
            assert [g[0] for g in got] == c["batches"]
            assert (st.page_fetches, st.page_reloads) == (c["page_fetches"], c["page_reloads"])
            want = list(O.loader_batches(path, c["batch_size"], c["order"], c["seed"], c["epoch"]))
            for (gi, gimg, glab), (wi, wa) in zip(got, want):
                assert gi == wi and np.array_equal(gimg, wa["image"]) and np.array_equal(glab, wa["label"])
    ds.close()


@pytest.mark.parametrize("chain", ["rrc:24,24|flip:0.5|normpc:1,2,3/4,5,6/f16", "crop:20,20|flip:0.5|normalize:3,2"])
def test_pool_stream_across_epochs_vs_oracle(tmp_path, chain):
    """Random order, a pool far smaller than the heap: most batches evict pages
    the same batch already read (deferred recycling), slots are reused across
    batches and epochs (iterate_steps), variable image sizes and RLE payloads."""
    path = tmp_path / "var.bbox"
    bx.write_dataset(bx.SyntheticImageSource(400, 40, 36, 3, seed=3), path,
                     bx.WriterConfig(seed=2, page_size=65536, compress_probability=0.4))
    ds = bx.open_dataset(path, bx.ProcessCacheStrategy(capacity_pages=18))
    cfg = bx.LoaderConfig(batch_size=16, order=bx.OrderKind.RANDOM, seed=11,
                          pipelines={"image": bx.parse_pipeline(chain)})
    spec = chain.replace("/f16", "|cast:f16")
    with bx.Loader(ds, cfg) as loader:
        got = [(list(b.indices), b["image"].cpu().numpy()) for b in loader.iterate_steps(60)]
    ds.close()
    want = []
    for e in range(3):
        want += list(O.loader_batches(path, 16, "random", 11, e, pipelines={"image": spec}))
    for (gi, gimg), (wi, wa) in zip(got, want[:60]):
        assert gi == wi and np.array_equal(gimg, wa["image"])


def test_direct_strategy_preads_with_latency(tmp_path):
    """Direct(read_latency_s) (reader.py:61-65,368-372): one counted pread per
    payload read, the latency spun first; batches identical to the oracle."""
    import time

    path = tmp_path / "d.bbox"
    bx.write_dataset(bx.SyntheticImageSource(64, 24, 20, 3, seed=4), path,
                     bx.WriterConfig(seed=1, page_size=65536, compress_probability=0.5))
    lat = 0.002
    ds = bx.open_dataset(path, bx.Direct(read_latency_s=lat))
    assert ds.io_read_count == 1
    cfg = bx.LoaderConfig(batch_size=16, order=bx.OrderKind.RANDOM, seed=5,
                          pipelines={"image": bx.parse_pipeline("crop:16,16|flip:0.5")})
    t0 = time.perf_counter()
    with bx.Loader(ds, cfg) as loader:
        got = [(list(b.indices), b["image"].cpu().numpy()) for b in loader.iterate_epoch(0)]
    el = time.perf_counter() - t0
    assert ds.io_read_count == 1 + 64
    assert el >= 64 * lat / (os_cpu := __import__("os").cpu_count() or 1)   # spun on the staging threads
    want = list(O.loader_batches(path, 16, "random", 5, 0, pipelines={"image": "crop:16,16|flip:0.5"}))
    for (gi, gimg), (wi, wa) in zip(got, want):
        assert gi == wi and np.array_equal(gimg, wa["image"])
    before = ds.io_read_count
    s = ds.get_sample(3)
    assert ds.io_read_count == before + 1 and np.array_equal(s["image"], O.decode(*_cell4(ds, 3)))
    ds.close()


def _cell4(ds, i):
    c = ds.cells(i)[0]
    raw = np.frombuffer(open(ds.path, "rb").read()[c.offset:c.offset + c.length], dtype=np.uint8)
    return c.height, c.width, c.channels, c.codec, raw
