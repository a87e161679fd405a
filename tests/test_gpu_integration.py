"""INTEGRATION.md's binding, run for real: integration/bbox_gpu.py drives libbbx
from the UNMODIFIED reference package (baseline/_ref, `pip install --target`):
its LoaderConfig, its Decode / RandomCrop / RandomFlip / Resize / Normalize /
ToFloat instances from its own parse_pipeline, its TraversalOrder.  Batches must
equal the reference Loader's golden batches (tests/golden/loader_batches.npz)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
GOLDEN = ROOT / "tests" / "golden"
CASES = [c for c in json.loads((GOLDEN / "loader_cases.json").read_text())["cases"]
         if c["dataset"] in ("tiny", "paged", "synth_rle") and c["fields"] is None]


@pytest.fixture(scope="module")
def ref():
    if not (REF / "bbox").exists():
        pytest.skip("baseline/_ref (the pip-installed reference) is not present")
    for p in (str(REF), str(ROOT)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import bbox
    from integration import bbox_gpu

    return bbox, bbox_gpu


@pytest.mark.parametrize("case", range(len(CASES)), ids=[f"{c['dataset']}-{c['case']}-e{c['epoch']}" for c in CASES])
def test_reference_api_through_libbbx(ref, case):
    bbox, bbox_gpu = ref
    c = CASES[case]
    cfg = c["config"]
    path = GOLDEN / f"{c['dataset']}.bbox"
    pipes = {k: bbox.parse_pipeline(v) for k, v in c["pipelines"].items()}
    config = bbox.LoaderConfig(batch_size=cfg["batch_size"], order=bbox.OrderKind(cfg["order"]),
                               seed=cfg.get("seed", 0), drop_last=cfg.get("drop_last", False), pipelines=pipes or None)
    ds = bbox.open_dataset(path)
    page_map = ([ds.primary_page(i) for i in range(ds.num_samples)]
                if config.order == bbox.OrderKind.QUASI_RANDOM else None)
    batches = bbox.TraversalOrder(config.order, config.seed).epoch_batches(
        c["epoch"], ds.num_samples, config.batch_size, page_map, config.drop_last)
    ds.close()
    gl = bbox_gpu.GpuLoader(path, config)
    try:
        got = [(list(b.indices), b.arrays["image"].cpu().numpy(), b.arrays["label"].cpu().numpy())
               for b in gl.iterate_epoch(batches, c["epoch"])]
    finally:
        gl.close()
    data = np.load(GOLDEN / "loader_batches.npz")
    assert len(got) == c["num_batches"]
    for bi, (gi, gimg, glab) in enumerate(got):
        k = f"{c['key']}/b{bi}"
        assert gi == data[k + "/indices"].tolist()
        assert np.array_equal(gimg, data[k + "/image"])
        assert np.array_equal(glab, data[k + "/label"])
