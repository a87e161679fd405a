"""Sample sources for the writer (fixtures and bench data).

Same contracts as sources.py:51-159 of the reference: `schema`, `len()`,
integer indexing.  SyntheticImageSource content is a pure function of
(seed, i): label = below(num_classes), base = below(256) from stream
(seed, TAG_SYNTH, i); pixel (y, x, c) = (base + 11y + 3(x >> 2) + 7c) & 255.
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np

from .errors import SchemaMismatch, SourceError
from .format import array_field, image_field, int_field
from .rng import TAG_SYNTH, Rng, stream_seed

RASTER_HEADER = struct.Struct("<III")
RASTER_EXT = ".raw"


class InMemorySource:
    def __init__(self, schema, samples):
        self.schema = list(schema)
        self._samples = list(samples)

    def __len__(self) -> int:
        return len(self._samples)

    def __getitem__(self, i: int) -> dict:
        return self._samples[i]


class SyntheticImageSource:
    def __init__(self, num_samples: int, height: int = 32, width: int = 32, channels: int = 3, seed: int = 0,
                 num_classes: int = 10):
        self.num_samples = num_samples
        self.height, self.width, self.channels = height, width, channels
        self.seed = seed
        self.num_classes = num_classes
        self.schema = [image_field("image", height, width, channels), int_field("label")]
        yy = np.arange(height, dtype=np.int64).reshape(-1, 1, 1) * 11
        xx = (np.arange(width, dtype=np.int64) >> 2).reshape(1, -1, 1) * 3
        cc = np.arange(channels, dtype=np.int64).reshape(1, 1, -1) * 7
        self._pattern = ((yy + xx + cc) & 0xFF).astype(np.uint8)

    def __len__(self) -> int:
        return self.num_samples

    def _draws(self, i: int) -> tuple[int, int]:
        r = Rng(stream_seed(self.seed, TAG_SYNTH, i))
        return r.below(self.num_classes), r.below(256)

    def label_of(self, i: int) -> int:
        return self._draws(i)[0]

    def __getitem__(self, i: int) -> dict:
        if not 0 <= i < self.num_samples:
            raise IndexError(i)
        label, base = self._draws(i)
        # u8 wrap-around add == (pattern + base) & 255
        return {"image": self._pattern + np.uint8(base), "label": label}


class PhotoLikeSource:
    """ImageNet-shaped synthetic photos for the JPEG configs (bench data and fixtures).

    Not a reference source (the reference's SyntheticImageSource pattern is too
    smooth for JPEG: SURVEY.md §8d).  Sample i is a pure function of (seed, i):
    size (h, w) with the longer side = max dims and the shorter one drawn in
    [min_frac, 1] x max (like an ImageNet file resized to max_res), a diagonal
    gradient with per-sample offsets, plus uniform noise of +-`noise`.
    Optional `array_dim` adds the sparse-regression case study's float32
    NDArray field "x" of that length (BASELINE configs[4]).
    """

    def __init__(self, num_samples: int, max_height: int = 256, max_width: int = 256, channels: int = 3,
                 seed: int = 0, num_classes: int = 1000, noise: int = 12, min_frac: float = 0.6,
                 fixed_size: bool = False, array_dim: int = 0):
        self.num_samples = num_samples
        self.max_height, self.max_width, self.channels = max_height, max_width, channels
        self.seed, self.num_classes, self.noise = seed, num_classes, noise
        self.min_frac, self.fixed_size, self.array_dim = min_frac, fixed_size, array_dim
        self.schema = [image_field("image", max_height, max_width, channels), int_field("label")]
        if array_dim:
            self.schema.append(array_field("x", np.float32, (array_dim,)))
        # shared gradient + noise bank (built once: __getitem__ runs on writer threads)
        yy = np.arange(max_height, dtype=np.int32)[:, None, None]
        xx = np.arange(max_width, dtype=np.int32)[None, :, None]
        cc = np.arange(channels, dtype=np.int32)[None, None, :]
        self._pattern = ((yy * (1 + cc) // 2 + xx * (3 - cc) // 2 + cc * 40) & 0xFF).astype(np.uint8)
        g = np.random.default_rng([seed, 0x5EED])
        nb = max_height * max_width * channels + (1 << 16)
        self._noise = g.integers(-noise, noise + 1, size=nb, dtype=np.int16).astype(np.int8).view(np.uint8)

    def __len__(self) -> int:
        return self.num_samples

    def dims_of(self, i: int) -> tuple[int, int]:
        if self.fixed_size:
            return self.max_height, self.max_width
        r = Rng(stream_seed(self.seed, TAG_SYNTH, i, 1))
        frac = self.min_frac + (1.0 - self.min_frac) * (r.below(1 << 20) / float(1 << 20))
        if r.below(2):
            return self.max_height, max(1, int(self.max_width * frac))
        return max(1, int(self.max_height * frac)), self.max_width

    def _tables(self):
        return self._pattern, self._noise

    def __getitem__(self, i: int) -> dict:
        if not 0 <= i < self.num_samples:
            raise IndexError(i)
        r = Rng(stream_seed(self.seed, TAG_SYNTH, i))
        label = r.below(self.num_classes)
        base = np.array([r.below(256) for _ in range(self.channels)], dtype=np.uint8)
        off = r.below(1 << 16)
        h, w = self.dims_of(i)
        pattern, noise = self._tables()
        img = pattern[:h, :w] + base                           # u8 wrap-around arithmetic
        if self.noise:
            img += noise[off:off + h * w * self.channels].reshape(h, w, self.channels)
        out = {"image": img, "label": label}
        if self.array_dim:
            out["x"] = np.random.default_rng([self.seed, i]).standard_normal(self.array_dim, dtype=np.float32)
        return out


def write_raster(path, pixels) -> None:
    px = np.asarray(pixels, dtype=np.uint8)
    if px.ndim != 3:
        raise SchemaMismatch("raster pixels must be HxWxC")
    with open(path, "wb") as fh:
        fh.write(RASTER_HEADER.pack(*px.shape))
        fh.write(np.ascontiguousarray(px).tobytes())


def read_raster(path) -> np.ndarray:
    with open(path, "rb") as fh:
        head = fh.read(RASTER_HEADER.size)
        if len(head) < RASTER_HEADER.size:
            raise SourceError(f"{path}: truncated raster header")
        h, w, c = RASTER_HEADER.unpack(head)
        data = fh.read(h * w * c)
    if len(data) != h * w * c:
        raise SourceError(f"{path}: raster payload truncated")
    return np.frombuffer(data, dtype=np.uint8).reshape(h, w, c).copy()


class DirectoryImageSource:
    """``root/<label>/<file>.raw`` trees (sorted labels, sorted files)."""

    def __init__(self, root):
        self.root = Path(root)
        self.label_names = sorted(p.name for p in self.root.iterdir() if p.is_dir())
        self.entries = []
        mh = mw = 0
        ch = None
        for li, name in enumerate(self.label_names):
            for f in sorted((self.root / name).glob(f"*{RASTER_EXT}")):
                with open(f, "rb") as fh:
                    head = fh.read(RASTER_HEADER.size)
                if len(head) < RASTER_HEADER.size:
                    raise SourceError(f"{f}: truncated raster header")
                h, w, c = RASTER_HEADER.unpack(head)
                if ch is None:
                    ch = c
                elif ch != c:
                    raise SourceError(f"{f}: mixed channel counts ({c} vs {ch})")
                mh, mw = max(mh, h), max(mw, w)
                self.entries.append((f, li))
        if not self.entries:
            raise SourceError(f"{self.root}: no {RASTER_EXT} files found")
        self.schema = [image_field("image", mh, mw, ch), int_field("label")]

    def __len__(self) -> int:
        return len(self.entries)

    def __getitem__(self, i: int) -> dict:
        path, label = self.entries[i]
        return {"image": read_raster(path), "label": label}


def materialize_to_directory(source, root) -> Path:
    root = Path(root)
    digits = max(len(str(max(len(source) - 1, 0))), 1)
    for i in range(len(source)):
        s = source[i]
        d = root / str(s["label"])
        os.makedirs(d, exist_ok=True)
        write_raster(d / f"{i:0{digits}d}{RASTER_EXT}", s["image"])
    return root
