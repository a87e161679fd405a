"""GPU parity at the exact shapes bench.py times (BASELINE.json configs[1..4]).

The column-walker K1 is persistent (SMs x resident CTAs, 592 on a B200) and
hands out tiles from a global ticket in runs; the smaller parity tests launch
fewer tiles than CTAs.  Here each launch has thousands of tiles (configs[1]:
512 samples x 12 tiles of 16 rows = 6,144), so every CTA takes several ticket
runs, the geometry ring wraps across samples and the column table is rebuilt
and re-copied between ring entries -- the regime the headline number runs in.
The JPEG legs use the bench writer's files (q90 4:2:0, a restart marker every
2 MCUs, batch 1024).  Each case streams across an epoch boundary with
iterate_steps (no pipeline drain), like the timed region does, and every batch
is compared bit for bit with the oracle (oracle/bbx_oracle.c, pinned to the
reference's goldens and to Pillow in tests/test_oracle.py).
"""

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O
from test_gpu_parity import assert_same, oracle_spec, to_np

pytestmark = pytest.mark.gpu

NORM = "normpc:123.675,116.28,103.53/58.395,57.12,57.375"
RRC192 = f"rrc:192,192|flip:0.5|{NORM}/f16"          # bench.py CHAIN_SPEC
RRC160 = f"rrc:160,160|flip:0.5|{NORM}/f16"
VAL224 = f"center:224,224,{224 / 256}|{NORM}/f16"   # bench.py VAL_SPEC
SEED = 3


def _gpu_steps(path, batch, order, steps, pipelines, strategy=None, start_epoch=0):
    pipes = {k: bx.parse_pipeline(v) for k, v in pipelines.items()}
    ds = bx.open_dataset(path, strategy)
    cfg = bx.LoaderConfig(batch_size=batch, order=bx.OrderKind(order), seed=SEED, pipelines=pipes)
    out = []
    with bx.Loader(ds, cfg) as loader:
        for b in loader.iterate_steps(steps, start_epoch=start_epoch):
            out.append((list(b.indices), {k: to_np(v) for k, v in b.arrays.items()}))
    ds.close()
    return out


def _oracle_steps(path, batch, order, steps, pipelines, start_epoch=0):
    spec = {k: oracle_spec(v) for k, v in pipelines.items()}
    out, epoch = [], start_epoch
    while len(out) < steps:
        out += list(O.loader_batches(path, batch, order, SEED, epoch, pipelines=spec, nthreads=16))
        epoch += 1
    return out[:steps]


@pytest.fixture(scope="module")
def raw256(tmp_path_factory):
    """configs[1]: the bench's SyntheticImageSource 256x256x3 RAW file (+ label)."""
    path = tmp_path_factory.mktemp("bench") / "imagenet256_raw_1280.bbox"
    bx.write_dataset(bx.SyntheticImageSource(1280, 256, 256, 3, seed=1), path, bx.WriterConfig(seed=1))
    return path


@pytest.fixture(scope="module")
def jpeg256(tmp_path_factory):
    """configs[2]/[3]: the bench's PhotoLikeSource JPEG q90 4:2:0, RST every 2 MCUs."""
    path = tmp_path_factory.mktemp("bench") / "imagenet256_jpeg_2100.bbox"
    bx.write_dataset(bx.PhotoLikeSource(2100, 256, 256, 3, seed=1), path,
                     bx.WriterConfig(seed=1, compress_probability=1.0, compress_codec=bx.CodecId.JPEG,
                                     jpeg=bx.JpegParams(90, "4:2:0", restart_blocks=2), num_encode_workers=8))
    return path


@pytest.mark.parametrize("resident", [True, False])
def test_configs1_raw_rrc192_batch512(raw256, resident):
    """1280 samples at batch 512: 512, 512, 256 (epoch 0), then 512 of epoch 1."""
    pipes = {"image": RRC192}
    strategy = bx.DeviceResident(0) if resident else None
    got = _gpu_steps(raw256, 512, "random", 4, pipes, strategy)
    want = _oracle_steps(raw256, 512, "random", 4, pipes)
    assert [len(i) for i, _ in got] == [512, 512, 256, 512]
    assert_same(got, want)


def test_configs1_raw_rrc160_batch512(raw256):
    pipes = {"image": RRC160}
    got = _gpu_steps(raw256, 512, "random", 3, pipes, bx.DeviceResident(0), start_epoch=2)
    assert_same(got, _oracle_steps(raw256, 512, "random", 3, pipes, start_epoch=2))


@pytest.mark.parametrize("resident", [True, False])
def test_configs2_jpeg_rrc192_batch1024(jpeg256, resident):
    """2100 samples at batch 1024: 1024, 1024, 52 (epoch 0), then 1024 of epoch 1."""
    pipes = {"image": RRC192}
    strategy = bx.DeviceResident(0) if resident else None
    got = _gpu_steps(jpeg256, 1024, "random", 4, pipes, strategy)
    want = _oracle_steps(jpeg256, 1024, "random", 4, pipes)
    assert [len(i) for i, _ in got] == [1024, 1024, 52, 1024]
    assert_same(got, want)


def test_configs2_jpeg_rrc160_batch1024(jpeg256):
    pipes = {"image": RRC160}
    got = _gpu_steps(jpeg256, 1024, "random", 2, pipes, bx.DeviceResident(0), start_epoch=1)
    assert_same(got, _oracle_steps(jpeg256, 1024, "random", 2, pipes, start_epoch=1))


def test_configs3_jpeg_center224_sequential(jpeg256):
    pipes = {"image": VAL224}
    got = _gpu_steps(jpeg256, 1024, "sequential", 3, pipes)
    assert_same(got, _oracle_steps(jpeg256, 1024, "sequential", 3, pipes))


def test_configs4_jpeg_quasi_ndarray(tmp_path):
    """configs[4]: quasi-random JPEG RRC-192 + a float32 NDArray (d = 50,000) at batch 1024."""
    path = tmp_path / "jpeg_nd.bbox"
    bx.write_dataset(bx.PhotoLikeSource(1100, 256, 256, 3, seed=1, array_dim=50000), path,
                     bx.WriterConfig(seed=1, compress_probability=1.0, compress_codec=bx.CodecId.JPEG,
                                     jpeg=bx.JpegParams(90, "4:2:0", restart_blocks=2), num_encode_workers=8))
    pipes = {"image": RRC192}
    got = _gpu_steps(path, 1024, "quasi-random", 3, pipes)
    want = _oracle_steps(path, 1024, "quasi-random", 3, pipes)
    assert [len(i) for i, _ in got] == [1024, 76, 1024]
    assert_same(got, want)
    assert got[0][1]["x"].dtype == np.float32 and got[0][1]["x"].shape == (1024, 50000)
