"""Golden vectors for the JPEG codec extension (codec id 3).

The reference has no JPEG codec (codecs.py:25-28), so parity for JPEG decode
is anchored on the third-party decoder FFCV uses, libjpeg-turbo, as shipped
in this image through Pillow 12.2.  This script encodes a sweep of images
with Pillow (sizes incl. odd / tiny ones, 4:2:0 / 4:2:2 / 4:4:4 / grayscale,
quality 50/90/100, restart intervals none / 1 / 2 MCU rows and 3 MCUs) and
stores the JPEG bytes with Pillow's decoded pixels.  The oracle
(oracle/jpeg_oracle.c) must reproduce these bit for bit
(tests/test_oracle.py::test_jpeg_oracle_matches_pillow_goldens), and the
device decoder must match the oracle (tests/test_gpu_jpeg.py).

Run from the repo root:  python tests/golden/make_jpeg_golden.py
"""

from __future__ import annotations

import hashlib
import io
import json
from pathlib import Path

import numpy as np
from PIL import Image, features

OUT = Path(__file__).resolve().parent


def photo(h, w, c, seed, noise=12):
    g = np.random.default_rng(seed)
    yy = np.arange(h)[:, None, None]
    xx = np.arange(w)[None, :, None]
    cc = np.arange(c)[None, None, :]
    img = g.integers(0, 256, size=c)[None, None, :] + yy * (1 + cc) // 2 + xx * (3 - cc) // 2 + cc * 40
    img = img + g.integers(-noise, noise + 1, size=(h, w, c))
    return (img & 0xFF).astype(np.uint8)


def encode(px, quality, subsampling, rst_rows=0, rst_blocks=0):
    c = px.shape[2]
    im = Image.fromarray(px[:, :, 0] if c == 1 else px, "L" if c == 1 else "RGB")
    kw = {"quality": quality}
    if c == 3:
        kw["subsampling"] = subsampling
    if rst_rows:
        kw["restart_marker_rows"] = rst_rows
    if rst_blocks:
        kw["restart_marker_blocks"] = rst_blocks
    bio = io.BytesIO()
    im.save(bio, "JPEG", **kw)
    return bio.getvalue()


def pillow_decode(b, c):
    a = np.asarray(Image.open(io.BytesIO(b)).convert("L" if c == 1 else "RGB"))
    return a[:, :, None] if c == 1 else a


def main():
    cases = []
    seed = 0
    sizes = [(1, 1), (2, 3), (8, 8), (9, 17), (16, 16), (17, 9), (31, 33), (40, 64), (5, 70), (64, 48)]
    for h, w in sizes:
        for c, ss in [(3, "4:2:0"), (3, "4:2:2"), (3, "4:4:4"), (1, None)]:
            for q, rr, rb in [(90, 1, 0), (50, 0, 0), (100, 2, 0), (90, 0, 3)]:
                seed += 1
                px = photo(h, w, c, seed)
                b = encode(px, q, ss, rr, rb)
                cases.append(dict(h=h, w=w, c=c, ss=ss, q=q, rst_rows=rr, rst_blocks=rb, jpeg=b,
                                  pix=pillow_decode(b, c)))
    big = []
    for i, (h, w, ss) in enumerate([(256, 256, "4:2:0"), (256, 181, "4:2:0"), (203, 256, "4:4:4"),
                                    (256, 256, "4:2:2")]):
        px = photo(h, w, 3, 1000 + i)
        b = encode(px, 90, ss, 1)
        big.append(dict(h=h, w=w, c=3, ss=ss, q=90, jpeg=b,
                        sha256=hashlib.sha256(pillow_decode(b, 3).tobytes()).hexdigest()))
    blob = b"".join(c["jpeg"] for c in cases) + b"".join(c["jpeg"] for c in big)
    offs = np.cumsum([0] + [len(c["jpeg"]) for c in cases] + [len(c["jpeg"]) for c in big])
    pix = np.concatenate([c["pix"].reshape(-1) for c in cases])
    poffs = np.cumsum([0] + [c["pix"].size for c in cases])
    np.savez_compressed(OUT / "jpeg_cases.npz", jpeg=np.frombuffer(blob, np.uint8), offs=offs, pix=pix,
                        poffs=poffs)
    meta = {
        "generator": "Pillow %s, libjpeg-turbo %s" % (Image.__version__, features.version("libjpeg_turbo")),
        "small": [{k: v for k, v in c.items() if k not in ("jpeg", "pix")} for c in cases],
        "big": [{k: v for k, v in c.items() if k != "jpeg"} for c in big],
    }
    (OUT / "jpeg_cases.json").write_text(json.dumps(meta, indent=1))
    print(f"{len(cases)} small + {len(big)} big cases, {len(blob)} JPEG bytes")


if __name__ == "__main__":
    main()
