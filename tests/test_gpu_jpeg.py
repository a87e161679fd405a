"""GPU parity for the JPEG codec extension (codec id 3): the device decoder
(csrc/jpeg.cu through the C ABI) against the pinned oracle
(oracle/jpeg_oracle.c == Pillow/libjpeg-turbo, tests/test_oracle.py).

Tolerance: none.  north_star allows +-1 LSB for JPEG decode and bilinear
resize; this decoder restates libjpeg-turbo's integer arithmetic (ISLOW IDCT,
fancy upsampling, fixed-point color), so decoded pixels and every chain on
top of them are compared bit for bit.
"""

import hashlib

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O
from test_gpu_parity import assert_same, oracle_spec, run_gpu

pytestmark = pytest.mark.gpu


def test_decode_image_matches_oracle_and_pillow_goldens(golden):
    import torch

    for m, jpeg, px, sha in O.jpeg_golden_cases(golden):
        out = torch.empty((m["h"], m["w"], m["c"]), dtype=torch.uint8, device="cuda")
        bx.decode_image(bx.ImageBlob(m["h"], m["w"], m["c"], bx.CodecId.JPEG, jpeg), out)
        got = out.cpu().numpy()
        want = O.decode(m["h"], m["w"], m["c"], 3, jpeg)
        assert np.array_equal(got, want), m
        if px is not None:
            assert np.array_equal(got, px), m
        else:
            assert hashlib.sha256(got.tobytes()).hexdigest() == sha, m


def _jpeg_dataset(tmp_path, n=96, side=64, channels=3, subsampling="4:2:0", restart_rows=1, p=1.0, quality=90,
                  seed=1, fixed=False):
    src = bx.PhotoLikeSource(n, side, side, channels, seed=seed, fixed_size=fixed, min_frac=0.3)
    path = tmp_path / f"jpeg_{channels}_{subsampling.replace(':', '')}_{restart_rows}_{p}.bbox"
    bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 20, seed=seed, compress_probability=p,
                                                compress_codec=bx.CodecId.JPEG,
                                                jpeg=bx.JpegParams(quality, subsampling, restart_rows=max(restart_rows, 0),
                                                                   restart_blocks=-restart_rows if restart_rows < 0 else 0)))
    return path


JPEG_CHAINS = [
    "decode",
    "rrc:40,40|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16",
    "rrc:17,31,0.3,1,0.5,2|flip:0.5|normalize:127.5,64",
    "center:56,56,0.875|normpc:123.675,116.28,103.53/58.395,57.12,57.375/bf16",
    "crop:48,40|flip:0.5|normpc:1,2,3/4,5,6/f32",
]


# restart: > 0 every that many MCU rows, < 0 every -n MCUs, 0 none
@pytest.mark.parametrize("layout", [("4:2:0", 1), ("4:2:2", 2), ("4:4:4", 0), ("4:2:0", 0), ("4:2:0", -3), ("4:4:4", -1)])
@pytest.mark.parametrize("chain", JPEG_CHAINS)
def test_jpeg_chains_vs_oracle(tmp_path, layout, chain):
    path = _jpeg_dataset(tmp_path, subsampling=layout[0], restart_rows=layout[1])
    got = run_gpu(path, 20, "random", seed=17, epoch=1, pipelines={"image": chain})
    want = list(O.loader_batches(path, 20, "random", 17, 1, pipelines={"image": oracle_spec(chain)}, nthreads=4))
    assert_same(got, want)


def test_jpeg_grayscale_and_mixed_codecs_vs_oracle(tmp_path):
    for channels, p in ((1, 1.0), (3, 0.5)):
        path = _jpeg_dataset(tmp_path, n=70, side=48, channels=channels, p=p, seed=5)
        chain = "rrc:32,32|flip:0.5|normalize:127.5,64"
        got = run_gpu(path, 16, "quasi-random", seed=3, epoch=0, pipelines={"image": chain})
        want = list(O.loader_batches(path, 16, "quasi-random", 3, 0, pipelines={"image": chain}))
        assert_same(got, want)


def test_jpeg_imagenet_shape_resident_and_staged(tmp_path):
    """configs[2]-shaped batch (256-side, 4:2:0, RRC-192 f16) through every payload
    path: staged, HBM-resident, and a pinned heap (zero_copy requested: JPEG plans
    stage from it, csrc/engine.cpp finalize)."""
    path = _jpeg_dataset(tmp_path, n=80, side=256, seed=9)
    chain = "rrc:192,192|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16"
    want = list(O.loader_batches(path, 40, "random", 3, 0, pipelines={"image": oracle_spec(chain)}, nthreads=8))
    for strategy in (None, bx.DeviceResident(), bx.OsCache(zero_copy=True)):
        got = run_gpu(path, 40, "random", seed=3, epoch=0, pipelines={"image": chain}, strategy=strategy)
        assert_same(got, want)


def _cell(path, i):
    f = O.OracleFile(path)
    off, length, h, w, c, codec = f.cell(i, f.fields[0])
    return dict(offset=off, length=length, h=h, w=w, c=c, codec=codec)


def _corrupt_copy(path, out, i, fn):
    raw = bytearray(path.read_bytes())
    c = _cell(path, i)
    fn(raw, c)
    out.write_bytes(bytes(raw))
    return c


def _first_error(path, bs):
    ds = bx.open_dataset(path)
    loader = bx.Loader(ds, bx.LoaderConfig(batch_size=bs, order=bx.OrderKind.SEQUENTIAL))
    seen = []
    try:
        with pytest.raises(bx.errors.CorruptPayload) as ei:
            for b in loader.iterate_epoch(0):
                seen += list(b.indices)
    finally:
        loader.shutdown()
        ds.close()
    return seen, str(ei.value)


def test_jpeg_corrupt_payloads_raise_at_their_position(tmp_path):
    path = _jpeg_dataset(tmp_path, n=12, side=64, seed=2, fixed=True)

    def break_soi(raw, c):                       # host-detected (header parse)
        raw[c["offset"]] = 0x00

    def swap_rst(raw, c):                        # device-detected (J1 marker sequence)
        seg = bytes(raw[c["offset"]:c["offset"] + c["length"]])
        j = seg.find(b"\xff\xd1")
        assert j > 0
        raw[c["offset"] + j + 1] = 0xD5

    for i, fn, msg in ((5, break_soi, "SOI"), (9, swap_rst, "restart marker")):
        bad = tmp_path / f"bad{i}.bbox"
        c = _corrupt_copy(path, bad, i, fn)
        for bs in (4, 3):
            seen, err = _first_error(bad, bs)
            assert msg in err, err
            assert seen == list(range(i // bs * bs))
        with pytest.raises(O.OracleError):
            O.decode(c["h"], c["w"], c["c"], 3, bad.read_bytes()[c["offset"]:c["offset"] + c["length"]])


def test_configs4_shape_distributed_slices_vs_oracle(tmp_path):
    """configs[4] shape: JPEG RRC + float32 NDArray field, QUASI_RANDOM order,
    distributed=True with 2 ranks: the ranks' slices concatenate to the oracle's
    global batch (images bit-exact, array rows exact, labels exact)."""
    src = bx.PhotoLikeSource(90, 64, 64, 3, seed=4, min_frac=0.4, array_dim=300)
    path = tmp_path / "c4.bbox"
    bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 18, seed=4, compress_probability=1.0,
                                                compress_codec=bx.CodecId.JPEG))
    chain = "rrc:48,48|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16"
    parts = [run_gpu(path, 8, "quasi-random", seed=9, epoch=1, pipelines={"image": chain}, distributed=True,
                     rank=r, world_size=2) for r in range(2)]
    glob = list(O.loader_batches(path, 16, "quasi-random", 9, 1, pipelines={"image": oracle_spec(chain)}))
    assert len(parts[0]) == len(glob)
    for g, (gi, ga) in enumerate(glob):
        idx, arrs = [], {k: [] for k in ga}
        for r in range(2):
            if g < len(parts[r]):
                idx += parts[r][g][0]
                for k in ga:
                    arrs[k].append(parts[r][g][1][k])
        assert idx == gi
        for k in ga:
            assert np.array_equal(np.concatenate(arrs[k]), ga[k]), k


def test_repeated_epochs_are_deterministic(tmp_path):
    """Regression for a staging-pool race (a late worker could claim indices of the
    next parallel_for and skip payload copies): the same epoch, run repeatedly through
    the staged path with a JPEG field + an NDArray field, must not change."""
    src = bx.PhotoLikeSource(90, 64, 64, 3, seed=4, min_frac=0.4, array_dim=300)
    path = tmp_path / "det.bbox"
    bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 18, seed=4, compress_probability=1.0,
                                                compress_codec=bx.CodecId.JPEG))
    chain = "rrc:48,48|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16"
    ref = run_gpu(path, 8, "quasi-random", seed=9, epoch=1, pipelines={"image": chain})
    for _ in range(6):
        assert_same(run_gpu(path, 8, "quasi-random", seed=9, epoch=1, pipelines={"image": chain}), ref)
    for i, (_, arrs) in enumerate(ref):
        assert np.array_equal(arrs["x"], np.stack([src[j]["x"] for j in ref[i][0]]))


def test_unsupported_jpeg_processes_raise_at_their_position(tmp_path):
    """A progressive JPEG cell (SOF2) and a non-JPEG payload in a JPEG field are
    rejected host-side with CorruptPayload at the sample's position; the oracle
    rejects the same bytes."""
    import io

    from PIL import Image

    src = bx.PhotoLikeSource(10, 40, 40, 3, seed=6, fixed_size=True)
    path = tmp_path / "p.bbox"
    bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 16, seed=6, compress_probability=1.0,
                                                compress_codec=bx.CodecId.JPEG))
    raw = bytearray(path.read_bytes())
    c = _cell(path, 6)
    bio = io.BytesIO()
    Image.fromarray(src[6]["image"]).save(bio, "JPEG", quality=90, progressive=True)
    prog = bio.getvalue()
    assert len(prog) <= c["length"]
    raw[c["offset"]:c["offset"] + len(prog)] = prog
    bad = tmp_path / "prog.bbox"
    bad.write_bytes(bytes(raw))
    with pytest.raises(O.OracleError, match="progressive"):
        O.decode(c["h"], c["w"], c["c"], 3, prog)
    for bs in (4, 5):
        seen, err = _first_error(bad, bs)
        assert "progressive" in err, err
        assert seen == list(range(6 // bs * bs))
