"""GPU parity of the CUDA-graph replay path (engine.cpp process_slot: a full
HBM-resident batch without per-sample device status is captured once per
(slot, compute stream) and replayed): many batches over a few slots, so every
slot's graph is replayed several times with new descriptors, bit-exact against
the oracle and against the same loader with graphs off."""

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O
from test_gpu_parity import oracle_spec, to_np

pytestmark = pytest.mark.gpu

NORM = "normpc:123.675,116.28,103.53/58.395,57.12,57.375"


def _dataset(tmp_path, n=48, side=40):
    rs = np.random.default_rng(5)
    schema = [bx.image_field("image", side, side, 3), bx.int_field("label")]
    samples = []
    for i in range(n):
        img = rs.integers(0, 256, size=(side, side, 3), dtype=np.uint8)
        samples.append({"image": img, "label": 1000 + i})
    path = tmp_path / "graphs.bbox"
    bx.write_dataset(bx.InMemorySource(schema, samples), path, bx.WriterConfig(page_size=1 << 16, seed=5))
    return path


def _run(path, chain, steps, batch, slots, graphs):
    ds = bx.open_dataset(path, bx.DeviceResident(0))
    cfg = bx.LoaderConfig(batch_size=batch, order=bx.OrderKind.RANDOM, seed=9, slot_count=slots,
                          pipelines={"image": bx.parse_pipeline(chain)}, options={"cuda_graphs": int(graphs)})
    out = []
    with bx.Loader(ds, cfg) as loader:
        for b in loader.iterate_steps(steps, start_epoch=2):
            out.append((list(b.indices), {k: to_np(v) for k, v in b.arrays.items()}))
    ds.close()
    return out


@pytest.mark.parametrize("chain", [f"rrc:24,24|flip:0.5|{NORM}/f16",       # column-walker K1
                                   "flip:0.5|normalize:127.5,64"])            # tile K1 + prologue
def test_graph_replay_matches_oracle(tmp_path, chain):
    path = _dataset(tmp_path)
    batch, per_epoch, epochs = 8, 6, 4
    got = _run(path, chain, per_epoch * epochs, batch, 3, graphs=True)
    off = _run(path, chain, per_epoch * epochs, batch, 3, graphs=False)
    want = []
    for e in range(2, 2 + epochs):
        want += list(O.loader_batches(path, batch, "random", 9, e, pipelines={"image": oracle_spec(chain)}))
    assert len(got) == len(off) == len(want) == per_epoch * epochs
    for k, ((gi, ga), (oi, oa), (wi, wa)) in enumerate(zip(got, off, want)):
        assert gi == oi == list(wi), k
        for f in ("image", "label"):
            assert np.array_equal(ga[f], wa[f]), (k, f)
            assert np.array_equal(oa[f], wa[f]), (k, f)


def test_graph_replay_with_partial_batches(tmp_path):
    """50 samples in batches of 8: six full (graph) batches and a short one (plain
    launches) per epoch, interleaved on the same slots across epochs."""
    path = _dataset(tmp_path, n=50)
    chain = f"rrc:16,20|flip:0.5|{NORM}/bf16"
    got = _run(path, chain, 7 * 3, 8, 4, graphs=True)
    want = []
    for e in range(2, 5):
        want += list(O.loader_batches(path, 8, "random", 9, e, pipelines={"image": oracle_spec(chain)}))
    assert len(got) == len(want) == 21
    for k, ((gi, ga), (wi, wa)) in enumerate(zip(got, want)):
        assert gi == list(wi), k
        for f in ("image", "label"):
            assert np.array_equal(ga[f], wa[f]), (k, f)
