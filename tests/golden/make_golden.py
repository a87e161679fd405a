"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here comes from the unmodified reference package `bbox`
(/root/reference/pkg/src/bbox): its writer produces the .bbox files, its
Loader produces the expected batches, its rng/traversal produce the KATs.
The tests compare the oracle restatement (oracle/) and the CUDA path against
these files; nothing in the product imports them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

import bbox
from bbox import (
    InMemorySource,
    Loader,
    LoaderConfig,
    OrderKind,
    SyntheticImageSource,
    WriterConfig,
    open_dataset,
    write_dataset,
)
from bbox import pipeline as pl
from bbox import rng as brng
from bbox.codecs import CodecId, ImageBlob, decode_image, encode_image
from bbox.format import array_field, bytes_field, float_field, image_field, int_field
from bbox.traversal import TraversalOrder

OUT = Path(__file__).resolve().parent
PAGE = 65536


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


# --------------------------------------------------------------------------- rng
def rng_kats() -> dict:
    out = {}
    r = brng.Rng(0)
    out["rng0_first3"] = [hex(r.next_u64()) for _ in range(3)]
    out["stream_seed"] = []
    for seed, parts in [(3, (2, 0, 0, 0)), (3, (2, 0, 1, 0)), (3, (2, 0, 2, 0)),
                        (3, (2, 0, 3, 0)), (0, (1, 0)), (7, (1, 5)), (2**64 - 1, (4, 123456)),
                        (11, (2, 1, 199, 0)), (5, (3, 17))]:
        out["stream_seed"].append([seed, list(parts), hex(brng.stream_seed(seed, *parts))])
    out["below"] = []
    for seed, n in [(42, 17), (1, 1), (9, 1000003), (123, 2**40 + 7), (77, 65)]:
        r = brng.Rng(seed)
        out["below"].append([seed, n, [r.below(n) for _ in range(64)]])
    out["chance"] = []
    for seed, p in [(5, 0.5), (6, 0.25), (7, 0.999), (8, 1e-3), (9, 0.0), (10, 1.0), (11, 0.1)]:
        r = brng.Rng(seed)
        seq = [bool(r.chance(p)) for _ in range(64)]
        out["chance"].append([seed, p, seq, hex(r.state)])
    out["permutation"] = [[s, n, brng.permutation(s, n)] for s, n in [(7, 100), (8, 10), (0, 1), (1, 2)]]
    return out


# ----------------------------------------------------------------------- orders
def order_kats() -> dict:
    out = {"cases": []}
    rs = np.random.default_rng(2024)
    for kind in (OrderKind.SEQUENTIAL, OrderKind.RANDOM, OrderKind.QUASI_RANDOM):
        for (n, bs, seed, epoch, pages) in [
            (0, 4, 1, 0, None), (1, 3, 2, 0, None), (10, 4, 3, 1, "blocks5"),
            (200, 16, 4, 0, "blocks20"), (333, 7, 9, 2, "random"), (1000, 64, 3, 0, "withnone"),
            (97, 97, 5, 3, "blocks3"), (50, 128, 6, 0, "blocks8"),
        ]:
            if pages is None:
                pm = None
            elif pages == "random":
                pm = [int(x) for x in rs.integers(0, 40, size=n)]
            elif pages == "withnone":
                pm = [None if i % 13 == 0 else i // 37 for i in range(n)]
            else:
                k = int(pages[len("blocks"):])
                pm = [i // k for i in range(n)]
            order = TraversalOrder(kind, seed)
            for drop_last in (False, True):
                if kind == OrderKind.QUASI_RANDOM:
                    batches = order.epoch_batches(epoch, n, bs, pm, drop_last)
                else:
                    batches = order.epoch_batches(epoch, n, bs, pm, drop_last)
                out["cases"].append({
                    "kind": kind.value, "n": n, "batch_size": bs, "seed": seed, "epoch": epoch,
                    "page_map": pm, "drop_last": drop_last, "batches": batches,
                })
    return out


# --------------------------------------------------------------------- datasets
sys.path.insert(0, str(OUT))
from fixture_sources import dataset_builders  # noqa: E402

DATASETS = dataset_builders(bbox)

# (dataset, name, LoaderConfig kwargs, {field: pipeline spec}, fields, epochs)
LOADER_CASES = [
    ("tiny", "seq_default", dict(batch_size=6, order="sequential"), {}, None, [0]),
    ("tiny", "rand_crop_flip_norm", dict(batch_size=7, order="random", seed=5),
     {"image": "crop:6,6|flip:0.5|normalize:127.5,64"}, None, [0, 1]),
    ("tiny", "seq_drop_last", dict(batch_size=8, order="sequential", drop_last=True),
     {"image": "flip:1.0|float"}, None, [0]),
    ("paged", "rand_crop24", dict(batch_size=16, order="random", seed=11),
     {"image": "crop:24,24|flip:0.5|normalize:127.5,64"}, None, [0]),
    ("paged", "quasi_default", dict(batch_size=6, order="quasi-random", seed=4), {}, None, [0, 3]),
    ("paged", "seq_resize_crop", dict(batch_size=32, order="sequential", seed=2),
     {"image": "resize:40,20|crop:16,16|flip:0.25|float"}, None, [0]),
    ("paged", "rand_resize_down", dict(batch_size=50, order="random", seed=8),
     {"image": "resize:13,29|normalize:3,7"}, None, [1]),
    ("paged", "rand_norm_chain", dict(batch_size=64, order="random", seed=1),
     {"image": "flip:0.5|normalize:10,3|normalize:-1.5,0.3|crop:30,31"}, None, [0]),
    ("mixed_rle", "rand_all_fields", dict(batch_size=8, order="random", seed=2),
     {"image": "crop:10,10|flip:0.5|normalize:10,3"}, None, [0]),
    ("mixed_rle", "seq_default_all", dict(batch_size=16, order="sequential"), {}, None, [0]),
    ("mixed_rle", "quasi_arrays", dict(batch_size=5, order="quasi-random", seed=3),
     {"vec": "normalize:1,2", "patch": "crop:4,4|flip:0.5|float", "wide": "float",
      "ids": "normalize:0,1"}, ["vec", "patch", "wide", "ids", "label"], [0]),
    ("mixed_sub2", "rand_sub2", dict(batch_size=9, order="random", seed=13),
     {"image": "resize:16,16|crop:12,12|flip:0.5|float"}, None, [0]),
    ("mixed_sub2", "seq_sub2_decode", dict(batch_size=10, order="sequential"), {}, ["image", "score"], [0]),
    ("synth_rle", "rand_rle", dict(batch_size=12, order="random", seed=21),
     {"image": "crop:16,16|flip:0.5|normalize:127.5,64"}, None, [0]),
]


def parse_chain(spec: str):
    toks = [t for t in spec.split("|") if t]
    return pl.parse_pipeline("|".join(toks))


def run_loader(path, cfg_kwargs, pipelines, fields, epoch):
    cfg = dict(cfg_kwargs)
    cfg["order"] = OrderKind(cfg["order"])
    pipes = {k: parse_chain(v) for k, v in pipelines.items()} if pipelines else None
    loader = Loader(str(path), LoaderConfig(**cfg, pipelines=pipes, fields=fields))
    res = []
    try:
        for b in loader.iterate_epoch(epoch):
            res.append((list(map(int, b.indices)), {k: np.array(b[k], copy=True) for k in b.keys()}))
    finally:
        loader.shutdown()
    return res


def chain_vectors() -> dict:
    """Per-sample chain equivalence vectors (reference PipelinePlan)."""
    from bbox.format import ImageCell

    chains = [
        "decode", "decode|float", "decode|normalize:127.5,64", "decode|flip:0.5",
        "decode|crop:9,9", "decode|resize:6,14", "decode|crop:10,10|flip:0.5|normalize:10,3",
        "decode|resize:16,16|crop:12,12|flip:0.25|float", "decode|normalize:0,1",
        "decode|resize:25,7|normalize:-3.25,0.125", "decode|flip:0.5|flip:0.5|crop:3,12",
    ]
    rs = np.random.default_rng(999)
    arrays = {}
    meta = []
    for ci, spec in enumerate(chains):
        for trial in range(24):
            h = int(rs.integers(1, 13)) if trial % 2 else 12
            w = int(rs.integers(1, 13)) if trial % 2 else 12
            img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
            codec = CodecId(int(rs.integers(0, 3)))
            blob = encode_image(img, codec)
            cell = ImageCell(0, len(blob.payload), blob.height, blob.width, blob.channels, int(codec))
            seed = int(rs.integers(0, 2**63))
            p = pl.PipelinePlan(parse_chain(spec), pl.ImageSourceSpec(12, 12, 3), 1, 1)
            r = brng.Rng(seed)
            p.execute_sample((cell, np.frombuffer(blob.payload, dtype=np.uint8)), 0, 0, r)
            out = p.output_view(0, 1)[0].copy()
            key = f"c{ci}_t{trial}"
            arrays[key + "_payload"] = np.frombuffer(blob.payload, dtype=np.uint8).copy()
            arrays[key + "_out"] = out
            meta.append({"key": key, "chain": spec, "h": h, "w": w, "c": 3, "codec": int(codec),
                         "seed": hex(seed), "state_after": hex(r.state)})
    np.savez_compressed(OUT / "chains.npz", **arrays)
    return {"max": [12, 12, 3], "cases": meta}


def codec_error_vectors() -> dict:
    cases = []
    img = np.arange(64, dtype=np.uint8).reshape(8, 8, 1)
    rle = encode_image(img, CodecId.RLE).payload
    zero = bytearray(rle)
    zero[0:4] = (0).to_bytes(4, "little")
    over = bytearray(rle)
    over[0:4] = (1000).to_bytes(4, "little")
    blobs = [
        ("rle_truncated_run", 8, 8, 1, CodecId.RLE, rle[:-5]),
        ("rle_ragged", 8, 8, 1, CodecId.RLE, rle[:-2]),
        ("rle_zero_count", 8, 8, 1, CodecId.RLE, bytes(zero)),
        ("rle_overflow", 8, 8, 1, CodecId.RLE, bytes(over)),
        ("rle_empty", 8, 8, 1, CodecId.RLE, b""),
        ("raw_short", 2, 2, 1, CodecId.RAW, b"\x00" * 3),
        ("raw_long", 2, 2, 1, CodecId.RAW, b"\x00" * 5),
        ("sub2_short", 3, 3, 2, CodecId.SUBSAMPLE2, b"\x00" * 7),
        ("rle_ok", 8, 8, 1, CodecId.RLE, rle),
    ]
    for name, h, w, c, codec, payload in blobs:
        out = np.zeros((h, w, c), dtype=np.uint8)
        try:
            decode_image(ImageBlob(h, w, c, codec, payload), out)
            err = None
        except bbox.BboxError as e:
            err = [type(e).__name__, str(e)]
        cases.append({"name": name, "h": h, "w": w, "c": c, "codec": int(codec),
                      "payload": payload.hex(), "error": err, "out": out.tobytes().hex()})
    return {"cases": cases}


def corrupt_file_case() -> dict:
    """A reference-written RLE file with one payload corrupted on disk."""
    src = SyntheticImageSource(12, 6, 6, 3, seed=3)
    path = OUT / "corrupt_rle.bbox"
    write_dataset(src, path, WriterConfig(page_size=PAGE, seed=3, compress_probability=1.0))
    ds = open_dataset(path)
    victim = 7
    cell = ds.cells(victim)[0]
    ds.close()
    data = bytearray(path.read_bytes())
    data[cell.offset:cell.offset + 4] = (0).to_bytes(4, "little")  # zero-count run
    path.write_bytes(bytes(data))
    res = {"victim": victim}
    for bs in (4, 12):
        try:
            run_loader(path, dict(batch_size=bs, order="sequential"), {}, None, 0)
            res[f"bs{bs}"] = None
        except bbox.BboxError as e:
            res[f"bs{bs}"] = [type(e).__name__, str(e)]
    return res


def big_hashes() -> dict:
    """Per-batch sha256 of reference Loader output at bench-shaped configs.

    The .bbox files are regenerated on the GPU box by our own writer (checked
    byte-identical here via the file hash), then the CUDA loader's batches are
    hashed and compared with these.
    """
    tmp = Path(os.environ.get("GOLDEN_TMP", "/tmp/bbx_golden"))
    tmp.mkdir(parents=True, exist_ok=True)
    out = {}
    cases = [
        ("c1", dict(n=50_000, h=32, w=32, c=3, seed=1), {},
         dict(batch_size=512, order="random", seed=3), {"image": "flip:0.5|normalize:127.5,64"}, [0]),
        ("c2proxy", dict(n=1024, h=256, w=256, c=3, seed=1), {},
         dict(batch_size=512, order="random", seed=3), {"image": "crop:192,192|flip:0.5|normalize:127.5,64"}, [0]),
        ("c2resize", dict(n=600, h=256, w=256, c=3, seed=1), {},
         dict(batch_size=512, order="random", seed=3),
         {"image": "resize:224,224|crop:192,192|flip:0.5|normalize:127.5,64"}, [0]),
        ("rle64", dict(n=96, h=64, w=64, c=3, seed=2), dict(compress_probability=0.5),
         dict(batch_size=32, order="quasi-random", seed=3), {"image": "crop:48,48|flip:0.5|normalize:127.5,64"}, [0]),
    ]
    for name, src_kw, wkw, cfg, pipes, epochs in cases:
        path = tmp / f"{name}.bbox"
        src = SyntheticImageSource(src_kw["n"], src_kw["h"], src_kw["w"], src_kw["c"], seed=src_kw["seed"])
        write_dataset(src, path, WriterConfig(seed=src_kw["seed"], **wkw))
        entry = {"source": src_kw, "writer": wkw, "config": cfg, "pipelines": pipes,
                 "file_sha256": sha(path.read_bytes()), "epochs": {}}
        for e in epochs:
            batches = run_loader(path, cfg, pipes, None, e)
            entry["epochs"][str(e)] = [
                {"indices_sha256": sha(np.asarray(idx, dtype=np.int64).tobytes()),
                 "count": len(idx),
                 "image_sha256": sha(np.ascontiguousarray(arr["image"]).tobytes()),
                 "label_sha256": sha(np.ascontiguousarray(arr["label"]).tobytes())}
                for idx, arr in batches
            ]
            print(name, "epoch", e, len(batches), "batches", flush=True)
        out[name] = entry
    return out


def main() -> None:
    (OUT / "rng_kat.json").write_text(json.dumps(rng_kats(), indent=1))
    (OUT / "orders.json").write_text(json.dumps(order_kats()))
    files = {}
    for name, (builder, wkw) in DATASETS.items():
        path = OUT / f"{name}.bbox"
        src = builder()
        write_dataset(src, path, WriterConfig(**wkw))
        files[name] = {"sha256": sha(path.read_bytes()), "writer": {k: (int(v) if isinstance(v, CodecId) else v)
                                                                     for k, v in wkw.items()}}
    arrays = {}
    cases = []
    for ds_name, case, cfg, pipes, fields, epochs in LOADER_CASES:
        for e in epochs:
            batches = run_loader(OUT / f"{ds_name}.bbox", cfg, pipes, fields, e)
            key = f"{ds_name}/{case}/e{e}"
            for bi, (idx, arrs) in enumerate(batches):
                arrays[f"{key}/b{bi}/indices"] = np.asarray(idx, dtype=np.int64)
                for k, v in arrs.items():
                    arrays[f"{key}/b{bi}/{k}"] = v
            cases.append({"dataset": ds_name, "case": case, "config": cfg, "pipelines": pipes,
                          "fields": fields, "epoch": e, "num_batches": len(batches), "key": key})
    np.savez_compressed(OUT / "loader_batches.npz", **arrays)
    (OUT / "loader_cases.json").write_text(json.dumps({"files": files, "cases": cases}, indent=1))
    (OUT / "chains.json").write_text(json.dumps(chain_vectors(), indent=1))
    (OUT / "codec_errors.json").write_text(json.dumps(codec_error_vectors(), indent=1))
    (OUT / "corrupt_rle.json").write_text(json.dumps(corrupt_file_case(), indent=1))
    if "--no-big" not in sys.argv:
        (OUT / "big_hashes.json").write_text(json.dumps(big_hashes(), indent=1))


if __name__ == "__main__":
    main()
