"""Deterministic fixture sources shared by make_golden.py (run against the
reference package) and the tests (run against ours).  `api` is either
package: it must provide image_field/int_field/float_field/array_field/
bytes_field and InMemorySource."""

import numpy as np


def mixed_source(api, n: int, seed: int, max_side: int = 12):
    rs = np.random.default_rng(seed)
    schema = [
        api.image_field("image", max_side, max_side, 3),
        api.int_field("label"),
        api.float_field("score"),
        api.array_field("vec", np.float32, (2, 3)),
        api.array_field("ids", np.int64, (4,)),
        api.array_field("patch", np.uint8, (6, 6, 3)),
        api.array_field("wide", np.float64, (5,)),
        api.bytes_field("blob"),
    ]
    samples = []
    for i in range(n):
        h = int(rs.integers(1, max_side + 1))
        w = int(rs.integers(1, max_side + 1))
        if i % 3 == 0:  # flat regions -> short RLE payloads
            img = np.repeat(rs.integers(0, 4, size=(h, 1, 1), dtype=np.uint8), w, axis=1)
            img = np.repeat(img, 3, axis=2)
        else:
            img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        samples.append({
            "image": img,
            "label": int(rs.integers(-2**40, 2**40)),
            "score": float(rs.normal() * 1e3),
            "vec": (rs.normal(size=(2, 3)) * 100).astype(np.float32),
            "ids": rs.integers(-2**62, 2**62, size=4, dtype=np.int64),
            "patch": rs.integers(0, 256, size=(6, 6, 3), dtype=np.uint8),
            "wide": rs.normal(size=5) * 1e5,
            "blob": bytes(rs.integers(0, 256, size=int(rs.integers(0, 9)), dtype=np.uint8)),
        })
    return api.InMemorySource(schema, samples)


def dataset_builders(api):
    """name -> (source factory, WriterConfig kwargs) for the committed .bbox fixtures."""
    PAGE = 65536
    C = api.CodecId
    return {
        "tiny": (lambda: api.SyntheticImageSource(20, 8, 8, 1, seed=7), dict(page_size=PAGE, seed=7)),
        "paged": (lambda: api.SyntheticImageSource(200, 32, 32, 3, seed=1), dict(page_size=PAGE, seed=1)),
        "mixed_rle": (lambda: mixed_source(api, 60, 5), dict(page_size=PAGE, seed=9, compress_probability=0.5,
                                                            compress_codec=C.RLE)),
        "mixed_sub2": (lambda: mixed_source(api, 45, 6), dict(page_size=PAGE, seed=4, compress_probability=0.6,
                                                             compress_codec=C.SUBSAMPLE2)),
        "synth_rle": (lambda: api.SyntheticImageSource(48, 20, 24, 3, seed=2),
                      dict(page_size=PAGE, seed=2, compress_probability=0.5, compress_codec=C.RLE)),
    }
