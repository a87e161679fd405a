"""Run one GPU chain vs the oracle on the variable-size fixture (debug helper)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import tempfile
import numpy as np
import paper_2306_12517_b200 as bx
from test_gpu_parity import _variable_dataset, run_gpu, oracle_spec, assert_same
from oracle import oracle as O

chain = sys.argv[1]
codec = bx.CodecId(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
with tempfile.TemporaryDirectory() as td:
    path = _variable_dataset(Path(td), codec)
    got = run_gpu(path, 20, "random", seed=17, epoch=1, pipelines={"image": chain})
    want = list(O.loader_batches(path, 20, "random", 17, 1, pipelines={"image": oracle_spec(chain)}, nthreads=4))
    assert_same(got, want)
print("ok", chain, codec)
