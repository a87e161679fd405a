"""GPU parity of the persistent column-walker K1 (image_kernel.cuh
image_cw_kernel) against the oracle, at the shapes that exercise its
plan-time choices: stage-slot bounds that force fewer rows per tile (heavy
downscale), upscale from tiny sources, odd output widths (scalar store tails),
f32 / u8 / f16 outputs (each vector-store width), grids with fewer tiles than
persistent CTAs, and the HBM-resident heap."""

import numpy as np
import pytest

import paper_2306_12517_b200 as bx
from oracle import oracle as O
from test_gpu_parity import assert_same, oracle_spec, run_gpu

pytestmark = pytest.mark.gpu

NORM = "normpc:123.675,116.28,103.53/58.395,57.12,57.375"


def _raw_dataset(tmp_path, n, lo, hi, seed):
    rs = np.random.default_rng(seed)
    schema = [bx.image_field("image", hi, hi, 3), bx.int_field("label")]
    samples = []
    for i in range(n):
        h, w = int(rs.integers(lo, hi + 1)), int(rs.integers(lo, hi + 1))
        yy, xx = np.mgrid[0:h, 0:w]
        img = np.stack([(yy * 3 + xx * 5 + 40 * c) & 255 for c in range(3)], -1).astype(np.uint8)
        img ^= rs.integers(0, 32, size=img.shape, dtype=np.uint8)
        samples.append({"image": img, "label": i})
    path = tmp_path / f"raw_{lo}_{hi}_{seed}.bbox"
    bx.write_dataset(bx.InMemorySource(schema, samples), path, bx.WriterConfig(page_size=1 << 22, seed=seed))
    return path


CASES = [
    # (chain, n, min side, max side, batch)
    ("rrc:8,8|flip:0.5|normalize:127.5,64", 40, 160, 256, 16),           # ~32x downscale: 2 rows per tile
    (f"rrc:192,192|flip:0.5|{NORM}/f16", 24, 8, 24, 8),                   # 8-24x upscale
    (f"rrc:33,191,0.08,1,0.75,1.333|flip:0.5|{NORM}/f32", 30, 100, 256, 7),  # odd width, 16-B f32 stores
    ("center:191,97,0.875", 30, 120, 256, 5),                             # u8, odd width: scalar tails
    (f"rrc:7,5|{NORM}/bf16", 3, 64, 200, 1),                              # a few tiles per launch
    (f"center:224,224,0.875|{NORM}/f16", 20, 200, 256, 9),                # the validation chain
]


@pytest.mark.parametrize("resident", [False, True])
@pytest.mark.parametrize("chain,n,lo,hi,batch", CASES)
def test_column_walker_vs_oracle(tmp_path, chain, n, lo, hi, batch, resident):
    path = _raw_dataset(tmp_path, n, lo, hi, seed=n + lo)
    strategy = bx.DeviceResident(0) if resident else None
    got = run_gpu(path, batch, "random", seed=11, epoch=3, pipelines={"image": chain}, strategy=strategy)
    want = list(O.loader_batches(path, batch, "random", 11, 3, pipelines={"image": oracle_spec(chain)}, nthreads=4))
    assert_same(got, want)
