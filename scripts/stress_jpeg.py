"""Determinism stress: run the same JPEG loader epoch repeatedly and report any
batch whose output differs from the first run (races show up as rare diffs)."""
import sys, tempfile
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2306_12517_b200 as bx
from test_gpu_parity import run_gpu

td = Path(tempfile.mkdtemp())
order = sys.argv[1] if len(sys.argv) > 1 else "quasi-random"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
codec_p = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
src = bx.PhotoLikeSource(90, 64, 64, 3, seed=4, min_frac=0.4, array_dim=300)
path = td / "c4.bbox"
bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 18, seed=4, compress_probability=codec_p,
                                            compress_codec=bx.CodecId.JPEG))
want_x = {i: src[i]["x"] for i in range(90)}
chain = "rrc:48,48|flip:0.5|normpc:123.675,116.28,103.53/58.395,57.12,57.375/f16"
strat = (lambda: bx.DeviceResident()) if (len(sys.argv) > 4 and sys.argv[4] == "resident") else (lambda: None)
ref = run_gpu(path, 8, order, seed=9, epoch=1, pipelines={"image": chain}, strategy=strat())
bad = 0
for rep in range(reps):
    got = run_gpu(path, 8, order, seed=9, epoch=1, pipelines={"image": chain}, strategy=strat())
    for g, ((gi, ga), (ri, ra)) in enumerate(zip(got, ref)):
        for k in ra:
            if not np.array_equal(ga[k], ra[k]):
                rows = [j for j in range(len(gi)) if not np.array_equal(ga[k][j], ra[k][j])]
                bad += 1
                print("rep", rep, "batch", g, "field", k, "positions", rows, "samples", [gi[j] for j in rows])
                if k == "x":
                    for j in rows:
                        gx, rx = ga[k][j], ra[k][j]
                        same_as = [i for i, v in want_x.items() if np.array_equal(v, gx)]
                        nz = int((gx != rx).sum())
                        print("   ref ok", np.array_equal(rx, want_x[gi[j]]), "ndiff", nz, "first", int(np.argmax(gx != rx)),
                              "zeros", int((gx == 0).sum()), "equals sample", same_as, gx[:4], rx[:4])
import os
print("order", order, "reps", reps, "bad batches", bad, sys.argv[3:], os.environ.get("BBX_JPEG_CACHE"))
