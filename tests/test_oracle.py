"""Pin the CPU oracle against golden vectors from the real reference.

Every fixture under tests/golden/ was produced by the unmodified reference
package (tests/golden/make_golden.py).  If these pass, the oracle used by the
GPU parity tests restates the reference exactly.
"""

import ctypes
import json

import numpy as np
import pytest

from oracle import oracle as O


def test_rng_kats(golden):
    k = json.loads((golden / "rng_kat.json").read_text())
    st = ctypes.c_uint64(0)
    assert [hex(O.lib().or_next(ctypes.byref(st))) for _ in range(3)] == k["rng0_first3"]
    for seed, parts, want in k["stream_seed"]:
        arr = (ctypes.c_uint64 * len(parts))(*parts)
        assert hex(O.lib().or_stream_seed(seed, arr, len(parts))) == want
        assert hex(O.stream_seed(seed, *parts)) == want
    for seed, n, seq in k["below"]:
        st = ctypes.c_uint64(seed)
        assert [O.lib().or_below(ctypes.byref(st), n) for _ in range(64)] == seq
    for seed, p, seq, final in k["chance"]:
        st = ctypes.c_uint64(seed)
        assert [bool(O.lib().or_chance(ctypes.byref(st), p)) for _ in range(64)] == seq
        assert hex(st.value) == final
    for s, n, perm in k["permutation"]:
        a = np.arange(n, dtype=np.int64)
        st = ctypes.c_uint64(s)
        O.lib().or_shuffle(ctypes.byref(st), a.ctypes.data, n)
        assert a.tolist() == perm


def test_orders(golden):
    k = json.loads((golden / "orders.json").read_text())
    for c in k["cases"]:
        got = O.epoch_batches(c["kind"], c["seed"], c["epoch"], c["n"], c["batch_size"], c["page_map"],
                              c["drop_last"])
        assert got == c["batches"], c["kind"]


def test_codec_errors(golden):
    k = json.loads((golden / "codec_errors.json").read_text())
    for c in k["cases"]:
        payload = np.frombuffer(bytes.fromhex(c["payload"]), dtype=np.uint8)
        payload = np.ascontiguousarray(payload) if len(payload) else np.zeros(1, np.uint8)
        n = c["h"] * c["w"] * c["c"]
        out = np.zeros(n, dtype=np.uint8)

        class E(ctypes.Structure):
            _fields_ = [("code", ctypes.c_int), ("msg", ctypes.c_char * 256)]

        e = E()
        rc = O.lib().or_decode_image(c["h"], c["w"], c["c"], c["codec"], payload.ctypes.data,
                                     len(bytes.fromhex(c["payload"])), out.ctypes.data, ctypes.addressof(e))
        if c["error"] is None:
            assert rc == 0
            assert out.tobytes().hex() == c["out"]
        else:
            assert rc == 1
            assert O.ERR_NAMES[e.code] == c["error"][0]
            assert e.msg.decode() == c["error"][1]


def test_chain_vectors(golden):
    meta = json.loads((golden / "chains.json").read_text())
    data = np.load(golden / "chains.npz")
    mh, mw, mc = meta["max"]
    field = {"kind": "image", "max_h": mh, "max_w": mw, "channels": mc}
    for c in meta["cases"]:
        ops = O.parse_spec(c["chain"])
        payload = data[c["key"] + "_payload"]
        out, st = O.chain_one(ops, field, c["h"], c["w"], c["c"], c["codec"], payload, int(c["seed"], 16))
        want = data[c["key"] + "_out"]
        assert out.dtype == want.dtype and out.shape == want.shape, c["key"]
        assert np.array_equal(out, want), c["key"]
        assert hex(st) == c["state_after"], c["key"]


def _cases(golden):
    return json.loads((golden / "loader_cases.json").read_text())["cases"]


def test_loader_batches(golden):
    data = np.load(golden / "loader_batches.npz")
    for c in _cases(golden):
        cfg = c["config"]
        got = list(O.loader_batches(golden / f"{c['dataset']}.bbox", cfg["batch_size"], cfg["order"],
                                    cfg.get("seed", 0), c["epoch"], cfg.get("drop_last", False),
                                    c["pipelines"], c["fields"], nthreads=2))
        assert len(got) == c["num_batches"], c["key"]
        for bi, (idx, arrays) in enumerate(got):
            k = f"{c['key']}/b{bi}"
            assert idx == data[k + "/indices"].tolist()
            names = {n.split("/")[-1] for n in data.files if n.startswith(k + "/")} - {"indices"}
            assert set(arrays) == names, k
            for name, arr in arrays.items():
                want = data[f"{k}/{name}"]
                assert arr.dtype == want.dtype and arr.shape == want.shape, (k, name)
                assert np.array_equal(arr, want), (k, name)


def test_corrupt_file(golden):
    k = json.loads((golden / "corrupt_rle.json").read_text())
    for bs in (4, 12):
        with pytest.raises(O.OracleError) as ei:
            list(O.loader_batches(golden / "corrupt_rle.bbox", bs, "sequential"))
        kind, msg = k[f"bs{bs}"]
        assert O.ERR_NAMES[ei.value.code] == kind
        # loader.py:400-402 wraps as "sample {index} failed: {err}"
        assert f"sample {k['victim']} failed: {ei.value.msg}" == msg


def test_bilinear_decoders_vs_opencv():
    """Extension ops have no reference; pin the resample to OpenCV INTER_LINEAR (+-1 LSB)."""
    cv2 = pytest.importorskip("cv2")
    rs = np.random.default_rng(0)
    field = {"kind": "image", "max_h": 64, "max_w": 64, "channels": 3}
    for trial in range(60):
        h, w = int(rs.integers(8, 65)), int(rs.integers(8, 65))
        img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        if trial % 2:
            img = cv2.GaussianBlur(img, (5, 5), 2.0)
        oh, ow = int(rs.integers(4, 80)), int(rs.integers(4, 80))
        seed = int(rs.integers(0, 2**63))
        ops = O.parse_spec(f"rrc:{oh},{ow}")
        out, _ = O.chain_one(ops, field, h, w, 3, 0, img.reshape(-1), seed)
        # recover the window the oracle drew and resample it with OpenCV
        st = ctypes.c_uint64(seed)
        t, l, ch, cw = (ctypes.c_int() for _ in range(4))
        sc = (ctypes.c_double * 2)(0.08, 1.0)
        ra = (ctypes.c_double * 2)(3 / 4, 4 / 3)
        O.lib().or_rrc_window(ctypes.byref(st), h, w, sc, ra, ctypes.byref(t), ctypes.byref(l),
                              ctypes.byref(ch), ctypes.byref(cw))
        crop = np.ascontiguousarray(img[t.value:t.value + ch.value, l.value:l.value + cw.value])
        ref = cv2.resize(crop, (ow, oh), interpolation=cv2.INTER_LINEAR)
        diff = np.abs(out.astype(np.int32) - ref.astype(np.int32))
        assert diff.max() <= 1, (trial, diff.max())
    # center crop
    for trial in range(20):
        h, w = int(rs.integers(8, 65)), int(rs.integers(8, 65))
        img = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        out, _ = O.chain_one(O.parse_spec("center:24,24,0.875"), field, h, w, 3, 0, img.reshape(-1), 1)
        s = min(h, w)
        c = int(0.875 * s)
        t, l = (h - c) // 2, (w - c) // 2
        ref = cv2.resize(np.ascontiguousarray(img[t:t + c, l:l + c]), (24, 24), interpolation=cv2.INTER_LINEAR)
        assert np.abs(out.astype(np.int32) - ref.astype(np.int32)).max() <= 1


def test_casts_match_numpy():
    field = {"kind": "image", "max_h": 8, "max_w": 8, "channels": 3}
    rs = np.random.default_rng(1)
    img = rs.integers(0, 256, size=(8, 8, 3), dtype=np.uint8)
    base, _ = O.chain_one(O.parse_spec("decode|normpc:123.675,116.28,103.53/58.395,57.12,57.375"), field,
                          8, 8, 3, 0, img.reshape(-1), 0)
    want = (img.astype(np.float32) - np.float32([123.675, 116.28, 103.53])) / np.float32([58.395, 57.12, 57.375])
    assert np.array_equal(base, want)
    h16, _ = O.chain_one(O.parse_spec("decode|normpc:123.675,116.28,103.53/58.395,57.12,57.375|cast:f16"),
                         field, 8, 8, 3, 0, img.reshape(-1), 0)
    assert np.array_equal(h16, want.astype(np.float16))
    import torch
    b16, _ = O.chain_one(O.parse_spec("decode|normpc:123.675,116.28,103.53/58.395,57.12,57.375|cast:bf16"),
                         field, 8, 8, 3, 0, img.reshape(-1), 0)
    tb = torch.from_numpy(want).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(b16, tb)


# ------------------------------------------------------- JPEG codec extension
def test_jpeg_oracle_matches_pillow_goldens(golden):
    """oracle/jpeg_oracle.c == Pillow/libjpeg-turbo, 0 LSB, on every golden case."""
    import hashlib

    cases = O.jpeg_golden_cases(golden)
    assert len(cases) >= 100
    for m, jpeg, px, sha in cases:
        got = O.decode(m["h"], m["w"], m["c"], 3, jpeg)
        if px is not None:
            assert np.array_equal(got, px), m
        else:
            assert hashlib.sha256(got.tobytes()).hexdigest() == sha, m


def test_jpeg_oracle_rejects_bad_streams(golden):
    m, jpeg, _, _ = O.jpeg_golden_cases(golden)[20]
    with pytest.raises(O.OracleError, match="SOI"):
        O.decode(m["h"], m["w"], m["c"], 3, b"\x00\x01" + jpeg[2:])
    with pytest.raises(O.OracleError, match="cell says"):
        O.decode(m["h"] + 1, m["w"], m["c"], 3, jpeg)
    prog = bytearray(jpeg)
    i = prog.find(b"\xff\xc0")
    prog[i + 1] = 0xC2
    with pytest.raises(O.OracleError, match="progressive"):
        O.decode(m["h"], m["w"], m["c"], 3, bytes(prog))
