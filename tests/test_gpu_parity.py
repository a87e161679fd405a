"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
batches and against the pinned oracle.  Bit-exact everywhere: every op on
this path is integer/byte work or a single IEEE f32 subtract+divide."""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O

sys.path.insert(0, str(Path(__file__).parent / "golden"))
from fixture_sources import mixed_source  # noqa: E402

pytestmark = pytest.mark.gpu


def to_np(t):
    import torch

    t = t.detach()
    if t.dtype == torch.bfloat16:
        t = t.view(torch.int16)
        return t.cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def run_gpu(path, batch_size, order="random", seed=0, epoch=0, drop_last=False, pipelines=None, fields=None,
            strategy=None, **ext):
    pipes = {k: bx.parse_pipeline(v) for k, v in (pipelines or {}).items()} or None
    ds = bx.open_dataset(path, strategy)
    cfg = bx.LoaderConfig(batch_size=batch_size, order=bx.OrderKind(order), seed=seed, drop_last=drop_last,
                          pipelines=pipes, fields=fields, **ext)
    out = []
    with bx.Loader(ds, cfg) as loader:
        for b in loader.iterate_epoch(epoch):
            out.append((list(b.indices), {k: to_np(v) for k, v in b.arrays.items()}))
    ds.close()
    return out


def oracle_spec(spec: str) -> str:
    """Product grammar -> oracle grammar (normpc:m/s/f16 -> normpc:m/s|cast:f16)."""
    parts = []
    for p in spec.split("|"):
        if p.startswith("normpc:") and p.count("/") == 2:
            body, dt = p.rsplit("/", 1)
            parts += [body, f"cast:{dt}"]
        else:
            parts.append(p)
    return "|".join(parts)


def assert_same(got, want):
    assert len(got) == len(want)
    for (gi, ga), (wi, wa) in zip(got, want):
        assert gi == wi
        assert set(ga) == set(wa)
        for k in wa:
            assert ga[k].dtype == wa[k].dtype, (k, ga[k].dtype, wa[k].dtype)
            assert ga[k].shape == wa[k].shape, (k, ga[k].shape, wa[k].shape)
            if not np.array_equal(ga[k], wa[k]):
                bad = np.argwhere(ga[k] != wa[k])
                raise AssertionError(f"{k}: {len(bad)} mismatches, first at {bad[0].tolist()}: "
                                     f"{ga[k][tuple(bad[0])]} vs {wa[k][tuple(bad[0])]}")


# --------------------------------------------------- reference golden batches
def test_loader_batches_match_reference(golden):
    data = np.load(golden / "loader_batches.npz")
    for c in json.loads((golden / "loader_cases.json").read_text())["cases"]:
        cfg = c["config"]
        got = run_gpu(golden / f"{c['dataset']}.bbox", cfg["batch_size"], cfg["order"], cfg.get("seed", 0),
                      c["epoch"], cfg.get("drop_last", False), c["pipelines"], c["fields"])
        want = []
        for bi in range(c["num_batches"]):
            k = f"{c['key']}/b{bi}"
            names = {n.split("/")[-1] for n in data.files if n.startswith(k + "/")} - {"indices"}
            want.append((data[k + "/indices"].tolist(), {n: data[f"{k}/{n}"] for n in names}))
        assert_same(got, want)


@pytest.mark.parametrize("case", ["c1", "c2proxy", "c2resize", "rle64"])
def test_bench_shaped_batches_match_reference_hashes(golden, tmp_path, case):
    ref = json.loads((golden / "big_hashes.json").read_text())[case]
    s = ref["source"]
    path = tmp_path / f"{case}.bbox"
    bx.write_dataset(bx.SyntheticImageSource(s["n"], s["h"], s["w"], s["c"], seed=s["seed"]), path,
                     bx.WriterConfig(seed=s["seed"], **ref["writer"]))
    assert hashlib.sha256(path.read_bytes()).hexdigest() == ref["file_sha256"]
    cfg = ref["config"]
    for e, batches in ref["epochs"].items():
        got = run_gpu(path, cfg["batch_size"], cfg["order"], cfg["seed"], int(e), pipelines=ref["pipelines"])
        assert len(got) == len(batches)
        for (idx, arr), want in zip(got, batches):
            assert hashlib.sha256(np.asarray(idx, np.int64).tobytes()).hexdigest() == want["indices_sha256"]
            assert hashlib.sha256(np.ascontiguousarray(arr["image"]).tobytes()).hexdigest() == want["image_sha256"]
            assert hashlib.sha256(np.ascontiguousarray(arr["label"]).tobytes()).hexdigest() == want["label_sha256"]


def test_corrupt_payload_error_and_reuse(golden):
    k = json.loads((golden / "corrupt_rle.json").read_text())
    for bs in (4, 12):
        kind, msg = k[f"bs{bs}"]
        ds = bx.open_dataset(golden / "corrupt_rle.bbox")
        loader = bx.Loader(ds, bx.LoaderConfig(batch_size=bs, order=bx.OrderKind.SEQUENTIAL))
        with pytest.raises(getattr(bx.errors, kind)) as ei:
            for _ in loader.iterate_epoch(0):
                pass
        assert str(ei.value) == msg
        # the ring is reusable after a failed epoch (loader.py:213-217 semantics)
        loader2 = bx.Loader(ds, bx.LoaderConfig(batch_size=5, order=bx.OrderKind.SEQUENTIAL, fields=["label"]))
        assert sum(b.size for b in loader2.iterate_epoch(0)) == 12
        loader2.shutdown()
        loader.shutdown()
        ds.close()


# ------------------------------------------------------------- vs the oracle
def _variable_dataset(tmp_path, codec, n=96, max_side=64, seed=3):
    rs = np.random.default_rng(seed)
    schema = [bx.image_field("image", max_side, max_side, 3), bx.int_field("label")]
    samples = []
    for i in range(n):
        h, w = int(rs.integers(max_side // 4, max_side + 1)), int(rs.integers(max_side // 4, max_side + 1))
        img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        if i % 4 == 0:
            img[:, : w // 2] = img[:, :1]   # runs for RLE
        samples.append({"image": img, "label": i})
    path = tmp_path / f"var_{int(codec)}.bbox"
    bx.write_dataset(bx.InMemorySource(schema, samples), path,
                     bx.WriterConfig(page_size=1 << 20, seed=seed, compress_probability=0.6, compress_codec=codec))
    return path


EXT_CHAINS = [
    "rrc:24,24|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16",
    "rrc:17,31,0.3,1,0.5,2|flip:0.5|normalize:127.5,64",
    "center:20,20,0.875|normpc:123.675,116.28,103.53/58.395,57.12,57.375/bf16",
    "center:40,28,1.0",
    "crop:48,40|resize:33,17|flip:0.5|normpc:1,2,3/4,5,6/f32",
    "resize:96,80|crop:70,71|flip:0.5|float",
    "flip:0.5|crop:64,64|normalize:0.5,0.25|normalize:-3,7",
    "rrc:64,64,1,1,1,1|normalize:127.5,64",
]


@pytest.mark.parametrize("codec", [bx.CodecId.RLE, bx.CodecId.SUBSAMPLE2])
@pytest.mark.parametrize("chain", EXT_CHAINS)
def test_chains_vs_oracle(tmp_path, codec, chain):
    path = _variable_dataset(tmp_path, codec)
    got = run_gpu(path, 20, "random", seed=17, epoch=1, pipelines={"image": chain})
    want = list(O.loader_batches(path, 20, "random", 17, 1, pipelines={"image": oracle_spec(chain)}, nthreads=4))
    assert_same(got, want)


@pytest.mark.parametrize("zero_copy", [False, True])
def test_mixed_fields_vs_oracle(tmp_path, zero_copy):
    """RLE / RAW images, arrays and scalars in one loader; zero_copy requested on a
    plan with RLE payloads: the loader stages from the pinned heap instead."""
    path = tmp_path / "mixed.bbox"
    bx.write_dataset(mixed_source(bx, 120, 11, max_side=40), path,
                     bx.WriterConfig(page_size=65536, seed=1, compress_probability=0.5))
    pipes = {"image": "crop:30,33|flip:0.5|normpc:1,2,3/4,5,6/bf16", "vec": "normalize:1,2",
             "patch": "crop:4,5|flip:0.5|normalize:3,2", "wide": "float", "ids": "normalize:-5,3"}
    got = run_gpu(path, 13, "quasi-random", seed=5, epoch=2, pipelines=pipes,
                  strategy=bx.OsCache(zero_copy=True) if zero_copy else None)
    want = list(O.loader_batches(path, 13, "quasi-random", 5, 2,
                                 pipelines={k: oracle_spec(v) for k, v in pipes.items()}))
    assert_same(got, want)


# ------------------------------------------------------------ loader contract
def test_staging_threads_and_resident_invariance(golden):
    path = golden / "paged.bbox"
    pipes = {"image": "crop:24,24|flip:0.5|normalize:127.5,64"}
    a = run_gpu(path, 16, seed=11, pipelines=pipes, staging_threads=1)
    b = run_gpu(path, 16, seed=11, pipelines=pipes, staging_threads=8, slot_count=2)
    c = run_gpu(path, 16, seed=11, pipelines=pipes, strategy=bx.DeviceResident())
    assert_same(b, a)
    assert_same(c, a)


def test_exactly_once_and_lease_reuse(golden):
    ds = bx.open_dataset(golden / "paged.bbox")
    loader = bx.Loader(ds, bx.LoaderConfig(batch_size=7, order=bx.OrderKind.RANDOM, seed=5))
    seen, ptrs = [], set()
    for b in loader.iterate_epoch(0):
        seen += b.indices
        ptrs.add(b["image"].data_ptr())
    assert sorted(seen) == list(range(200))
    assert len(ptrs) <= 3
    assert loader.last_stats.batches == 29 and loader.last_stats.samples == 200
    loader.shutdown()
    loader.shutdown()
    with pytest.raises(bx.errors.ShutdownError):
        next(loader.iterate_epoch(1))
    ds.close()


def test_abandoned_epoch_then_fresh_epoch(golden):
    ds = bx.open_dataset(golden / "paged.bbox")
    loader = bx.Loader(ds, bx.LoaderConfig(batch_size=8, seed=2))
    for _ in loader.iterate_epoch(0):
        break
    assert loader.last_stats is not None
    n = sum(b.size for b in loader.iterate_epoch(1))
    assert n == 200
    loader.shutdown()
    ds.close()


def test_distributed_slices_union_is_global_batch(golden):
    path = golden / "paged.bbox"
    parts = [run_gpu(path, 6, "random", seed=3, distributed=True, rank=r, world_size=2) for r in range(2)]
    glob = list(O.loader_batches(path, 12, "random", 3))
    assert len(parts[0]) == len(glob)
    for g, (gi, ga) in enumerate(glob):
        idx = []
        imgs = []
        for r in range(2):
            if g < len(parts[r]):
                idx += parts[r][g][0]
                imgs.append(parts[r][g][1]["image"])
        assert idx == gi
        assert np.array_equal(np.concatenate(imgs), ga["image"])


def test_decode_image_on_device(golden):
    import torch

    for c in json.loads((golden / "codec_errors.json").read_text())["cases"]:
        blob = bx.ImageBlob(c["h"], c["w"], c["c"], bx.CodecId(c["codec"]), bytes.fromhex(c["payload"]))
        out = torch.zeros((c["h"], c["w"], c["c"]), dtype=torch.uint8, device="cuda")
        if c["error"] is None:
            bx.decode_image(blob, out)
            assert out.cpu().numpy().tobytes().hex() == c["out"]
        else:
            with pytest.raises(getattr(bx.errors, c["error"][0]), match=__import__("re").escape(c["error"][1])):
                bx.decode_image(blob, out)


def test_nchw_view_and_opaque_rejected(golden):
    import torch

    ds = bx.open_dataset(golden / "paged.bbox")
    pipes = {"image": [bx.Decode(), bx.RandomFlip(0.5), bx.NormalizeImage([1, 2, 3], [4, 5, 6], torch.float16),
                       bx.ToTorchImage()]}
    with bx.Loader(ds, bx.LoaderConfig(batch_size=10, pipelines=pipes)) as ld:
        b = next(iter(ld))
        assert b["image"].shape == (10, 3, 32, 32) and b["image"].is_contiguous(memory_format=torch.channels_last)
    with pytest.raises(bx.errors.SpecMismatch, match="opaque"):
        bx.Loader(ds, bx.LoaderConfig(batch_size=4, pipelines={"image": [bx.Opaque(lambda i, o, r: None)]}))
    ds.close()


@pytest.mark.parametrize("gather", [1, 0])
@pytest.mark.parametrize("chain", ["rrc:24,24|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16",
                                   "crop:48,40|resize:33,17|flip:0.5|normpc:1,2,3/4,5,6/f32",
                                   "center:40,28,1.0"])
def test_zero_copy_payloads_match_oracle(tmp_path, chain, gather):
    """OsCache(zero_copy=True): the batch's RAW windows come over PCIe from the
    pinned host heap -- gathered into HBM by host_gather_kernel (default) or read by
    K1 itself (option zc_gather=0) -- same batches as the oracle, PCIe bytes counted."""
    path = _variable_dataset(tmp_path, bx.CodecId.SUBSAMPLE2)
    raw = tmp_path / "raw.bbox"
    src = bx.SyntheticImageSource(70, 64, 64, 3, seed=2)
    bx.write_dataset(src, raw, bx.WriterConfig(page_size=1 << 18, seed=2))
    for p in (path, raw):
        got = run_gpu(p, 16, "random", seed=5, epoch=0, pipelines={"image": chain},
                      strategy=bx.OsCache(zero_copy=True), options={"zc_gather": gather})
        want = list(O.loader_batches(p, 16, "random", 5, 0, pipelines={"image": oracle_spec(chain)}))
        assert_same(got, want)
    ds = bx.open_dataset(raw, bx.OsCache(zero_copy=True))
    with bx.Loader(ds, bx.LoaderConfig(batch_size=16, pipelines={"image": bx.parse_pipeline(chain)},
                                       options={"zc_gather": gather})) as ld:
        for _ in ld.iterate_epoch(0):
            pass
        st = ld.stats()
    ds.close()
    assert st["zero_copy_bytes"] > 0 and st["h2d_bytes"] < st["zero_copy_bytes"]


@pytest.mark.parametrize("strategy", ["os", "resident", "zero_copy"])
def test_array_copy_kernel_alignments(tmp_path, strategy):
    """ArrayRead with no transform is a straight copy (array_copy_kernel: 16-B
    stores, source realigned per sample): odd lengths and every source
    misalignment, staged / HBM-resident / zero-copy payloads."""
    rs = np.random.default_rng(3)
    schema = [bx.array_field("a", np.uint8, (1001,)), bx.array_field("b", np.float32, (7, 111)),
              bx.array_field("c", np.int64, (3,)), bx.array_field("d", np.uint8, (17,)), bx.int_field("label")]
    samples = [{"a": rs.integers(0, 256, 1001, dtype=np.uint8), "b": rs.normal(size=(7, 111)).astype(np.float32),
                "c": rs.integers(-2**60, 2**60, 3, dtype=np.int64), "d": rs.integers(0, 256, 17, dtype=np.uint8),
                "label": i} for i in range(37)]
    path = tmp_path / "arrays.bbox"
    bx.write_dataset(bx.InMemorySource(schema, samples), path, bx.WriterConfig(page_size=65536, seed=1))
    strat = {"os": bx.OsCache(), "resident": bx.DeviceResident(), "zero_copy": bx.OsCache(zero_copy=True)}[strategy]
    got = run_gpu(path, 8, "random", seed=2, epoch=1, strategy=strat)
    want = list(O.loader_batches(path, 8, "random", 2, 1))
    assert_same(got, want)
