"""Deterministic byte-level corruptions of the committed .bbox fixtures, shared
by make_validate_golden.py (run against the reference validator) and
tests/test_validate.py (run against ours).  Each recipe maps the fixture's
bytes to a damaged copy; offsets come from the file's own header."""

import struct

PREFIX = struct.Struct("<8sIQHQQQQ2x")   # format.py:57-60 header prefix
DESC = 124


def _hdr(b: bytes):
    magic, ver, n, nf, page, dto, ho, ato = PREFIX.unpack_from(b, 0)
    widths = [struct.unpack_from("<I", b, PREFIX.size + k * DESC + 64 + 1 + 48)[0] for k in range(nf)]
    kinds = [b[PREFIX.size + k * DESC + 64] for k in range(nf)]
    return dict(n=n, nf=nf, page=page, dto=dto, ho=ho, ato=ato, widths=widths, kinds=kinds)


def _cell_off(b: bytes, sample: int, kind: int) -> int:
    h = _hdr(b)
    rw = sum(h["widths"])
    pos = 0
    for k, w in zip(h["kinds"], h["widths"]):
        if k == kind:
            return h["dto"] + sample * rw + pos
        pos += w
    raise KeyError(kind)


def bad_magic(b):
    return b"XXXXXXXX" + b[8:]


def bad_version(b):
    return b[:8] + struct.pack("<I", 2) + b[12:]


def short_prefix(b):
    return b[:40]


def codec_5(b):            # image cell codec byte (offset 21 in the 24-byte IMAGE cell)
    o = _cell_off(b, 3, 4) + 21
    return b[:o] + bytes([5]) + b[o + 1:]


def dims_too_big(b):
    o = _cell_off(b, 1, 4) + 16
    return b[:o] + struct.pack("<H", 60000) + b[o + 2:]


def channel_mismatch(b):
    o = _cell_off(b, 2, 4) + 20
    return b[:o] + bytes([b[o] + 1]) + b[o + 1:]


def dangling_image(b):
    o = _cell_off(b, 4, 4)
    return b[:o] + struct.pack("<Q", 17) + b[o + 8:]


def dangling_array(b):
    o = _cell_off(b, 0, 2)
    return b[:o] + struct.pack("<Q", 3) + b[o + 8:]


def truncated_alloc(b):
    h = _hdr(b)
    return b[:h["ato"] + 12]


def overlapping_regions(b):
    h = _hdr(b)
    count = struct.unpack_from("<Q", b, h["ato"])[0]
    if count < 2:
        return b
    o = h["ato"] + 8 + 16   # region 1's offset -> region 0's offset + 1
    r0 = struct.unpack_from("<Q", b, h["ato"] + 8)[0]
    return b[:o] + struct.pack("<Q", r0 + 1) + b[o + 8:]


def heap_not_paged(b):     # alloc table moved one byte later: heap length not a page multiple
    h = _hdr(b)
    hdr = bytearray(b[:PREFIX.size])
    struct.pack_into("<Q", hdr, 46, h["ato"] + 1)   # alloc_table_offset: prefix bytes 46..53
    return bytes(hdr) + b[PREFIX.size:h["ato"]] + b"\0" + b[h["ato"]:]


RECIPES = {
    "bad_magic": bad_magic, "bad_version": bad_version, "short_prefix": short_prefix, "codec_5": codec_5,
    "dims_too_big": dims_too_big, "channel_mismatch": channel_mismatch, "dangling_image": dangling_image,
    "truncated_alloc": truncated_alloc, "overlapping_regions": overlapping_regions, "heap_not_paged": heap_not_paged,
}
ARRAY_RECIPES = {"dangling_array": dangling_array}
FIXTURES = ["tiny", "paged", "mixed_rle", "mixed_sub2", "synth_rle"]
