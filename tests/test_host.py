"""CPU-only tests of the host side: writer byte-identity, native orders, the
C ABI (loads + exports + dataset parsing without a GPU), spec compilation,
error mapping.  No CUDA device needed."""

import ctypes
import hashlib
import json
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from paper_2306_12517_b200 import _lib, pipeline as pl
from paper_2306_12517_b200.errors import BadMagic, InvalidFile, SchemaMismatch, SpecMismatch
from paper_2306_12517_b200.rng import Rng, permutation, stream_seed
from oracle import oracle as O

sys.path.insert(0, str(Path(__file__).parent / "golden"))
from fixture_sources import dataset_builders  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def sha(b):
    return hashlib.sha256(b).hexdigest()


# ------------------------------------------------------------------ writer
@pytest.mark.parametrize("name", ["tiny", "paged", "mixed_rle", "mixed_sub2", "synth_rle"])
def test_writer_byte_identical_to_reference(golden, tmp_path, name):
    builder, wkw = dataset_builders(bx)[name]
    path = tmp_path / f"{name}.bbox"
    bx.write_dataset(builder(), path, bx.WriterConfig(**wkw))
    assert path.read_bytes() == (golden / f"{name}.bbox").read_bytes()


def test_writer_c1_full_size_hash(golden, tmp_path):
    """The bench-shaped C1 file (50k x 32x32x3) equals the reference writer's, by sha256."""
    ref = json.loads((golden / "big_hashes.json").read_text())["c1"]
    s = ref["source"]
    path = tmp_path / "c1.bbox"
    bx.write_dataset(bx.SyntheticImageSource(s["n"], s["h"], s["w"], s["c"], seed=s["seed"]), path,
                     bx.WriterConfig(seed=s["seed"]))
    assert sha(path.read_bytes()) == ref["file_sha256"]


def test_writer_rejects_bad_sources(tmp_path):
    schema = [bx.image_field("image", 4, 4, 1), bx.int_field("label")]
    with pytest.raises(bx.errors.DimsExceedMax if hasattr(bx, "errors") else Exception):
        bx.write_dataset(bx.InMemorySource(schema, [{"image": np.zeros((5, 4, 1), np.uint8), "label": 0}]),
                         tmp_path / "x.bbox")
    assert not (tmp_path / "x.bbox").exists()
    with pytest.raises(SchemaMismatch):
        bx.write_dataset(bx.InMemorySource(schema, [{"image": np.zeros((2, 2, 1), np.uint8)}]), tmp_path / "y.bbox")


# -------------------------------------------------------------------- rng
def test_python_rng_kats(golden):
    k = json.loads((golden / "rng_kat.json").read_text())
    r = Rng(0)
    assert [hex(r.next_u64()) for _ in range(3)] == k["rng0_first3"]
    for seed, parts, want in k["stream_seed"]:
        assert hex(stream_seed(seed, *parts)) == want
    for seed, p, seq, final in k["chance"]:
        r = Rng(seed)
        assert [r.chance(p) for _ in range(64)] == seq and hex(r.state) == final
    for s, n, perm in k["permutation"]:
        assert permutation(s, n) == perm


# ----------------------------------------------------------------- orders
def test_native_orders_match_reference(golden):
    k = json.loads((golden / "orders.json").read_text())
    for c in k["cases"]:
        order = bx.TraversalOrder(bx.OrderKind(c["kind"]), c["seed"])
        got = order.epoch_batches(c["epoch"], c["n"], c["batch_size"], c["page_map"], c["drop_last"])
        assert got == c["batches"], (c["kind"], c["n"], c["batch_size"])


def test_native_quasi_order_large_matches_oracle():
    rs = np.random.default_rng(5)
    n = 20000
    pm = (np.arange(n) // 37).astype(np.int64)
    pm[rs.integers(0, n, 300)] = -1
    for bs in (1, 16, 512):
        got = bx.TraversalOrder(bx.OrderKind.QUASI_RANDOM, 9).epoch_indices(2, n, pm, bs)
        want = O.epoch_indices("quasi-random", 9, 2, n, [None if p < 0 else int(p) for p in pm], bs)
        assert got == want


def test_quasi_trace_structure():
    from paper_2306_12517_b200.traversal import QuasiRandomTrace

    pm = [i // 10 for i in range(100)]
    tr = QuasiRandomTrace()
    bx.TraversalOrder(bx.OrderKind.QUASI_RANDOM, 3).epoch_indices(0, 100, pm, 4, trace=tr)
    assert sorted(tr.page_loads) == list(range(10)) and tr.max_buffered == 4


def test_uniformity_probe_centred():
    m = bx.uniformity_probe(bx.OrderKind.RANDOM, 200, 50, seed=1)
    assert abs(m.mean() - 99.5) < 1e-9 and m.std() < 20


# ------------------------------------------------------------------ C ABI
def _header_functions():
    text = (ROOT / "include" / "bbx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bbx_[a-z_]+)\s*\(", text)))


def test_c_abi_exports_every_declared_symbol():
    declared = _header_functions()
    assert len(declared) >= 20
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bbx_\w+)", out))
    assert set(declared) <= exported
    assert b"sm_100a" in _lib.lib().bbx_version()


def test_dataset_open_without_gpu(golden):
    ds = bx.open_dataset(golden / "mixed_rle.bbox")
    try:
        of = O.OracleFile(golden / "mixed_rle.bbox")
        assert ds.num_samples == of.num_samples == 60
        assert [f.name for f in ds.schema] == [f["name"] for f in of.fields]
        for i in (0, 7, 59):
            assert ds.primary_page(i) == of.primary_page(i)
        np.testing.assert_array_equal(ds.column("label"), [of.cell(i, of.fields[1]) for i in range(60)])
        info = _lib.FieldInfo()
        _lib.check(_lib.lib().bbx_dataset_field(ds.handle, 0, ctypes.byref(info)))
        assert info.name == b"image" and info.max_height == 12 and info.channels == 3
        row = (ctypes.c_uint8 * 256)()
        _lib.check(_lib.lib().bbx_dataset_row(ds.handle, 3, row, 256))
        assert bytes(row[:ds.header.row_width]) == ds.row_bytes(3)
        with pytest.raises(bx.errors.IndexOutOfRange):
            ds.row_bytes(60)
    finally:
        ds.close()


def test_open_errors(tmp_path, golden):
    bad = tmp_path / "bad.bbox"
    data = bytearray((golden / "tiny.bbox").read_bytes())
    data[:8] = b"NOTMAGIC"
    bad.write_bytes(bytes(data))
    with pytest.raises(InvalidFile, match="bad magic"):
        bx.open_dataset(bad)
    h = ctypes.c_void_p()
    assert _lib.lib().bbx_dataset_open(str(bad).encode(), ctypes.byref(h)) == 2   # BBX_BAD_MAGIC
    short = tmp_path / "short.bbox"
    short.write_bytes(b"FASTDS01")
    with pytest.raises(InvalidFile):
        bx.open_dataset(short)
    with pytest.raises(FileNotFoundError):
        bx.open_dataset(tmp_path / "missing.bbox")


# ------------------------------------------------------------------ specs
def test_compile_chain_spec_rules():
    spec = pl.ImageSourceSpec(32, 32, 3)
    c = pl.compile_chain(pl.parse_pipeline("decode|crop:24,24|flip:0.5|normalize:127.5,64"), spec)
    assert [o.kind for o in c.ops] == [_lib.OP_DECODE, _lib.OP_CROP, _lib.OP_FLIP, _lib.OP_NORMALIZE]
    assert c.specs[-1] == ((24, 24, 3), np.dtype(np.float32))
    with pytest.raises(SpecMismatch, match="cannot crop"):
        pl.compile_chain(pl.parse_pipeline("decode|crop:40,4"), spec)
    with pytest.raises(SpecMismatch, match="first transform"):
        pl.compile_chain([pl.ToFloat()], spec)
    with pytest.raises(SpecMismatch, match="opaque"):
        pl.compile_chain([pl.Decode(), pl.Opaque(lambda i, o, r: None)], spec)
    with pytest.raises(SpecMismatch):
        pl.Normalize(0, 0)
    with pytest.raises(SpecMismatch, match="unknown transform"):
        pl.parse_pipeline("decode|blur:3")
    rrc = pl.compile_chain(pl.parse_pipeline("rrc:16,16|flip|normpc:1,2,3/4,5,6/bf16"), spec)
    assert [o.kind for o in rrc.ops] == [_lib.OP_RRC, _lib.OP_FLIP, _lib.OP_NORMALIZE_PC, _lib.OP_CAST]
    arr = pl.ArraySourceSpec((2, 3), np.dtype("f4"))
    with pytest.raises(SpecMismatch, match="HxWxC"):
        pl.compile_chain([pl.ArrayRead(), pl.RandomFlip()], arr)


def test_sharding_rule_partitions_global_batches():
    from paper_2306_12517_b200.loader import shard_batches

    order = bx.TraversalOrder(bx.OrderKind.RANDOM, 3)
    for world in (1, 2, 4, 8):
        gb = order.epoch_batches(0, 1000, 16 * world)
        parts = [shard_batches(gb, r, world, 16) for r in range(world)]
        flat = sorted(i for p in parts for b in p for i in b)
        assert flat == list(range(1000))
        for g in range(len(gb)):
            union = [i for r in range(world) if g < len(parts[r]) for i in parts[r][g]]
            assert union == gb[g][:len(union)]


def test_jpeg_writer_is_worker_count_independent(tmp_path):
    """Parallel encoding keeps the file byte-identical (allocation stays sequential)."""
    import hashlib

    import paper_2306_12517_b200 as bx

    src = bx.PhotoLikeSource(40, 48, 48, 3, seed=2, array_dim=7)
    digests = []
    for workers in (1, 4):
        p = tmp_path / f"w{workers}.bbox"
        bx.write_dataset(src, p, bx.WriterConfig(page_size=1 << 16, seed=2, compress_probability=0.7,
                                                 compress_codec=bx.CodecId.JPEG, num_encode_workers=workers))
        digests.append(hashlib.sha256(p.read_bytes()).hexdigest())
    assert digests[0] == digests[1]


def test_jpeg_payloads_decode_with_the_oracle(tmp_path):
    """Every JPEG cell the writer produces is a baseline file with restart markers that
    the oracle decodes exactly as Pillow / libjpeg-turbo does."""
    import io

    import numpy as np
    from PIL import Image

    import paper_2306_12517_b200 as bx
    from oracle import oracle as O

    src = bx.PhotoLikeSource(12, 40, 56, 3, seed=3)
    p = tmp_path / "j.bbox"
    bx.write_dataset(src, p, bx.WriterConfig(page_size=1 << 16, compress_probability=1.0,
                                             compress_codec=bx.CodecId.JPEG))
    f = O.OracleFile(p)
    for i in range(12):
        off, length, h, w, c, codec = f.cell(i, f.fields[0])
        assert codec == 3
        payload = bytes(f.buf[off:off + length])
        assert b"\xff\xdd" in payload                      # DRI present
        got = O.decode(h, w, c, 3, payload)
        assert np.array_equal(got, np.asarray(Image.open(io.BytesIO(payload)).convert("RGB")))
