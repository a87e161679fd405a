"""validate_file: every structural invariant of a .bbox container.

Restates the reference validator (format.py:396-548: decode_alloc_table,
ValidationReport, check_alloc_regions, _find_region, validate_file) with the
same checks, the same order and the same violation texts, vectorised over the
row table with numpy instead of a Python loop per sample.  One extension: the
reference rejects every codec > 2 (format.py:542-543); this build's JPEG codec
(id 3) is accepted, and each JPEG payload gets the decoder's own host-side
check (libbbx `bbx_jpeg_check`: header, dims == the cell's, Huffman tables,
restart-marker count and sequence) -- a file that validates is a file the
device path decodes.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .errors import InvalidFile, InvalidHeader
from .format import (FORMAT_VERSION, HEADER_PREFIX, MAGIC, FieldKind, decode_alloc_table, decode_header,
                     header_byte_length)

CODEC_JPEG = 3


@dataclass
class ValidationReport:
    path: str
    violations: list

    @property
    def ok(self) -> bool:
        return not self.violations

    def __str__(self) -> str:
        if self.ok:
            return f"{self.path}: valid"
        lines = [f"{self.path}: {len(self.violations)} violation(s)"]
        lines += [f"  - {v}" for v in self.violations]
        return "\n".join(lines)


def check_alloc_regions(regions, header) -> list:
    """Structural checks on a decoded allocation table (format.py:428-458)."""
    bad = []
    page = header.page_size
    prev_end = prev = None
    for r in regions:
        if r.length == 0:
            bad.append(f"empty region at offset {r.offset}")
            continue
        if r.offset < header.heap_offset or r.offset + r.length > header.alloc_table_offset:
            bad.append(f"region ({r.offset}, {r.length}) outside heap bounds")
        if prev_end is not None and r.offset < prev_end:
            bad.append(f"overlapping regions: ({prev.offset}, {prev.length}) and ({r.offset}, {r.length})")
        if prev is not None and r.offset < prev.offset:
            bad.append(f"regions not sorted at offset {r.offset}")
        rel = r.offset - header.heap_offset
        if r.length <= page:
            if rel % page + r.length > page:
                bad.append(f"region ({r.offset}, {r.length}) crosses a page boundary")
        elif rel % page:
            bad.append(f"oversized region ({r.offset}, {r.length}) not page aligned")
        prev_end = r.offset + r.length
        prev = r
    for i, r in enumerate(regions):   # oversized regions own whole pages
        if r.length > page:
            span_end = r.offset + -(-r.length // page) * page
            if i + 1 < len(regions) and regions[i + 1].offset < span_end:
                bad.append(f"oversized region ({r.offset}, {r.length}) shares a page")
    return bad


def _in_region(starts: np.ndarray, ends: np.ndarray, off: np.ndarray, length: np.ndarray) -> np.ndarray:
    """Vectorised _find_region (format.py:461-473): the last region starting at
    or before `off` (binary search on the region starts, in table order) must
    hold [off, off + length)."""
    if len(starts) == 0:
        return np.zeros(len(off), dtype=bool)
    # bisect_right over the table as stored (the reference's binary search assumes sorted starts)
    lo = np.zeros(len(off), dtype=np.int64)
    hi = np.full(len(off), len(starts), dtype=np.int64)
    while True:
        act = lo < hi
        if not act.any():
            break
        mid = (lo + hi) // 2
        go = act & (starts[np.minimum(mid, len(starts) - 1)] <= off)
        lo = np.where(go, mid + 1, lo)
        hi = np.where(act & ~go, mid, hi)
    k = lo - 1
    ok = k >= 0
    kk = np.maximum(k, 0)
    return ok & (off >= starts[kk]) & (off + length <= ends[kk])


def _jpeg_check(buf, off: int, length: int, h: int, w: int, c: int):
    from . import _lib

    L = _lib.lib()
    view = np.frombuffer(buf, dtype=np.uint8, count=length, offset=off)
    rc = L.bbx_jpeg_check(h, w, c, view.ctypes.data_as(ctypes.c_void_p), length)
    return None if rc == 0 else _lib.last_error()


def validate_file(path) -> ValidationReport:
    """Check every structural invariant of a container file.  Returns a report;
    an empty violation list means the file is valid.  I/O errors raise OSError."""
    violations: list = []
    file_len = os.path.getsize(path)
    with open(path, "rb") as fh:
        prefix = fh.read(HEADER_PREFIX.size)
        if len(prefix) < HEADER_PREFIX.size:
            return ValidationReport(str(path), ["file shorter than header prefix"])
        try:
            magic, version, num_samples, num_fields, *_ = HEADER_PREFIX.unpack(prefix)
            if magic != MAGIC:
                return ValidationReport(str(path), [f"bad magic {magic!r}"])
            if version != FORMAT_VERSION:
                return ValidationReport(str(path), [f"unsupported version {version}"])
            fh.seek(0)
            header = decode_header(fh.read(header_byte_length(num_fields)))
        except InvalidHeader as e:
            return ValidationReport(str(path), [f"invalid header: {e}"])

        rw = header.row_width
        table_end = header.data_table_offset + header.num_samples * rw
        if table_end > header.heap_offset:
            violations.append("data table extends past heap_offset")
        if header.alloc_table_offset > file_len:
            violations.append("alloc_table_offset past end of file")
            return ValidationReport(str(path), violations)
        if (header.alloc_table_offset - header.heap_offset) % header.page_size:
            violations.append("heap length is not a whole number of pages")
        fh.seek(header.alloc_table_offset)
        try:
            regions = decode_alloc_table(fh.read(file_len - header.alloc_table_offset))
        except InvalidFile as e:
            violations.append(str(e))
            return ValidationReport(str(path), violations)
        violations += check_alloc_regions(regions, header)
        if table_end > header.heap_offset or header.num_samples == 0:
            return ValidationReport(str(path), violations)

        fh.seek(header.data_table_offset)
        table = np.frombuffer(fh.read(header.num_samples * rw), dtype=np.uint8).reshape(header.num_samples, rw)
        rstart = np.array([r.offset for r in regions], dtype=np.int64)
        rend = rstart + np.array([r.length for r in regions], dtype=np.int64)
        n = header.num_samples
        per_sample: list = []   # (sample, field position, check order, text)
        pos = 0
        jpeg_cells = []
        for fpos, f in enumerate(header.fields):
            cell = table[:, pos:pos + f.row_cell_width]
            pos += f.row_cell_width
            if f.kind == FieldKind.FIXED_ARRAY:
                off = np.ascontiguousarray(cell[:, 0:8]).view("<u8").reshape(n).astype(np.int64)
                bad = ~_in_region(rstart, rend, off, np.full(n, f.array_nbytes, dtype=np.int64))
                for i in np.flatnonzero(bad):
                    per_sample.append((int(i), fpos, 0, f"dangling heap reference (sample {i}, field {f.name!r})"))
            elif f.kind == FieldKind.VAR_BYTES:
                off = np.ascontiguousarray(cell[:, 0:8]).view("<u8").reshape(n).astype(np.int64)
                ln = np.ascontiguousarray(cell[:, 8:16]).view("<u8").reshape(n).astype(np.int64)
                bad = (ln != 0) & ~_in_region(rstart, rend, off, ln)
                for i in np.flatnonzero(bad):
                    per_sample.append((int(i), fpos, 0, f"dangling heap reference (sample {i}, field {f.name!r})"))
            elif f.kind == FieldKind.IMAGE:
                off = np.ascontiguousarray(cell[:, 0:8]).view("<u8").reshape(n).astype(np.int64)
                ln = np.ascontiguousarray(cell[:, 8:16]).view("<u8").reshape(n).astype(np.int64)
                hh = np.ascontiguousarray(cell[:, 16:18]).view("<u2").reshape(n).astype(np.int64)
                ww = np.ascontiguousarray(cell[:, 18:20]).view("<u2").reshape(n).astype(np.int64)
                cc = cell[:, 20].astype(np.int64)
                codec = cell[:, 21].astype(np.int64)
                dims = (hh > f.max_height) | (ww > f.max_width)
                chan = cc != f.channels
                unk = codec > CODEC_JPEG
                dang = (ln != 0) & ~_in_region(rstart, rend, off, ln)
                for i in np.flatnonzero(dims):
                    per_sample.append((int(i), fpos, 0,
                                       f"image dims exceed descriptor max (sample {i}, field {f.name!r})"))
                for i in np.flatnonzero(chan):
                    per_sample.append((int(i), fpos, 1, f"image channel mismatch (sample {i}, field {f.name!r})"))
                for i in np.flatnonzero(unk):
                    per_sample.append((int(i), fpos, 2, f"unknown codec {int(codec[i])} (sample {i})"))
                for i in np.flatnonzero(dang):
                    per_sample.append((int(i), fpos, 3, f"dangling heap reference (sample {i}, field {f.name!r})"))
                # codec 3: the decoder's host check on every in-bounds JPEG payload
                js = np.flatnonzero((codec == CODEC_JPEG) & ~dang & (ln > 0))
                jpeg_cells.append((fpos, f.name, js, off, ln, hh, ww, cc))
        if jpeg_cells:
            import mmap

            with mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ) as mm:
                for fpos, name, js, off, ln, hh, ww, cc in jpeg_cells:
                    for i in js:
                        err = _jpeg_check(mm, int(off[i]), int(ln[i]), int(hh[i]), int(ww[i]), int(cc[i]))
                        if err:
                            per_sample.append((int(i), fpos, 4,
                                               f"invalid jpeg payload (sample {i}, field {name!r}): {err}"))
        per_sample.sort(key=lambda t: t[:3])
        violations += [t[3] for t in per_sample]
    return ValidationReport(str(path), violations)
