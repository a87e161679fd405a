"""Debug helper: loader batches on JPEG datasets vs the oracle, per sample."""
import sys, tempfile
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2306_12517_b200 as bx
from oracle import oracle as O
from test_gpu_parity import run_gpu

td = Path(tempfile.mkdtemp())
for channels, p in ((1, 1.0), (3, 0.5)):
    src = bx.PhotoLikeSource(70, 48, 48, channels, seed=5, min_frac=0.3)
    path = td / f"d{channels}.bbox"
    bx.write_dataset(src, path, bx.WriterConfig(page_size=1 << 20, seed=5, compress_probability=p,
                     compress_codec=bx.CodecId.JPEG, jpeg=bx.JpegParams(90, "4:2:0", restart_rows=1, restart_blocks=0)))
    for chain in ("decode", "rrc:32,32|flip:0.5|normalize:127.5,64"):
        got = run_gpu(path, 16, "quasi-random", seed=3, epoch=0, pipelines={"image": chain})
        want = list(O.loader_batches(path, 16, "quasi-random", 3, 0, pipelines={"image": chain}))
        nb = 0
        for (gi, ga), (wi, wa) in zip(got, want):
            for j in range(len(gi)):
                if not np.array_equal(ga["image"][j], wa["image"][j]):
                    nb += 1
                    if nb <= 3:
                        f = O.OracleFile(path); c = f.cell(gi[j], f.fields[0])
                        print(channels, p, chain, "sample", gi[j], "pos", j, "cell", c[2:], "codec", c[5])
        print(channels, p, chain, "bad samples", nb)
