"""Debug helper: per-sample device JPEG decode vs the oracle on a small dataset."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2306_12517_b200 as bx
from oracle import oracle as O

ch = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1
src = bx.PhotoLikeSource(70, 48, 48, ch, seed=5, min_frac=0.3)
bad = 0
for i in range(70):
    px = src[i]["image"]
    b = bx.codecs.encode_jpeg(px, bx.JpegParams(90, "4:2:0", restart_rows=rows, restart_blocks=0))
    h, w, c = px.shape
    out = torch.empty((h, w, c), dtype=torch.uint8, device="cuda")
    bx.decode_image(bx.ImageBlob(h, w, c, bx.CodecId.JPEG, b), out)
    got = out.cpu().numpy()
    want = O.decode(h, w, c, 3, b)
    if not np.array_equal(got, want):
        bad += 1
        d = np.argwhere(got != want)
        print("sample", i, (h, w, c), "mismatches", len(d), "first", d[0].tolist(), got[tuple(d[0])], want[tuple(d[0])])
print("bad", bad)
