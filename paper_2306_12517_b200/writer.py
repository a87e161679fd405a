"""Dataset writer (offline; produces files byte-identical to the reference's).

Layout rules of writer.py:138-278: heap starts at the first page boundary
after the row table; blobs are bump-allocated into pages and never straddle
one; a blob larger than a page gets its own run of whole pages while the open
page stays open; the allocation table (sorted regions) follows the last page.
Codec choice per sample: Rng(stream_seed(seed, TAG_CODEC, i)).chance(p).

Allocation is sequential (one lane), so the file is independent of
`num_encode_workers`; with one worker this is exactly the reference's layout.
Pages are assembled in memory and written whole.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .codecs import CodecId, JpegParams, encode_image
from .errors import InvalidFile, SchemaMismatch, SourceError
from .format import (
    DEFAULT_PAGE_SIZE, MIN_PAGE_SIZE, DatasetHeader, FieldKind, ImageCell, Region, VarBytesCell,
    decode_alloc_table, decode_header, encode_alloc_table, encode_header, encode_row, header_byte_length,
    row_width,
)
from .rng import TAG_CODEC, Rng, stream_seed


@dataclass
class WriterConfig:
    page_size: int = DEFAULT_PAGE_SIZE
    num_encode_workers: int = 1
    compress_probability: float = 0.0
    compress_codec: CodecId = CodecId.RLE
    seed: int = 0
    jpeg: JpegParams = field(default_factory=JpegParams)   # used when compress_codec is JPEG

    def check(self) -> None:
        ps = self.page_size
        if ps < MIN_PAGE_SIZE or ps & (ps - 1):
            raise ValueError(f"page_size must be a power of two >= {MIN_PAGE_SIZE}")
        if self.num_encode_workers < 1:
            raise ValueError("num_encode_workers must be >= 1")
        if not 0.0 <= self.compress_probability <= 1.0:
            raise ValueError("compress_probability must be in [0, 1]")


@dataclass
class WriteReport:
    path: str
    num_samples: int
    num_pages: int
    bytes_written: int
    codec_counts: dict
    waste_fraction: float


class _PagedHeap:
    """Single-lane bump allocator that buffers the open page in memory."""

    def __init__(self, fd: int, heap_offset: int, page_size: int):
        self.fd, self.base, self.page = fd, heap_offset, page_size
        self.next_page = 0
        self.open_page = None
        self.cursor = 0
        self.buf = bytearray(page_size)
        self.regions: list[Region] = []

    def _flush(self) -> None:
        if self.open_page is not None:
            os.pwrite(self.fd, bytes(self.buf[: self.cursor]), self.base + self.open_page * self.page)

    def put(self, data) -> int:
        n = len(data)
        if n < 1:
            raise ValueError("allocation length must be >= 1")
        if n > self.page:                        # dedicated whole pages; open page stays open
            first = self.next_page
            self.next_page += -(-n // self.page)
            off = self.base + first * self.page
            os.pwrite(self.fd, data, off)
        else:
            if self.open_page is None or self.page - self.cursor < n:
                self._flush()
                self.open_page = self.next_page
                self.next_page += 1
                self.cursor = 0   # only buf[:cursor] is ever written back
            off = self.base + self.open_page * self.page + self.cursor
            self.buf[self.cursor:self.cursor + n] = data
            self.cursor += n
        self.regions.append(Region(off, n))
        return off

    def finish(self) -> list[Region]:
        self._flush()
        return sorted(self.regions)


def write_dataset(source, path, config: WriterConfig | None = None, schema=None) -> WriteReport:
    config = config or WriterConfig()
    config.check()
    schema = list(schema if schema is not None else source.schema)
    n = len(source)
    rw = row_width(schema)
    hlen = header_byte_length(len(schema))
    page = config.page_size
    heap_offset = -(-(hlen + n * rw) // page) * page
    if heap_offset <= hlen:
        heap_offset += page
    rows = bytearray(n * rw)
    counts = {c: 0 for c in CodecId}
    fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        heap = _PagedHeap(fd, heap_offset, page)
        def encode_sample(i):
            """Source read + image encode of sample i (no allocation: thread-safe)."""
            try:
                values = source[i]
            except Exception as e:
                raise SourceError(f"sample {i}: {e}") from e
            draw = Rng(stream_seed(config.seed, TAG_CODEC, i))
            out = []
            for f in schema:
                if f.name not in values:
                    raise SchemaMismatch(f"sample {i} missing field {f.name!r}")
                v = values[f.name]
                if f.kind == FieldKind.INT_SCALAR:
                    out.append(int(v))
                elif f.kind == FieldKind.FLOAT_SCALAR:
                    out.append(float(v))
                elif f.kind == FieldKind.FIXED_ARRAY:
                    arr = np.ascontiguousarray(v, dtype=f.array_dtype)
                    if arr.shape != tuple(f.array_dims):
                        raise SchemaMismatch(f"sample {i} field {f.name!r}: shape {arr.shape} != {f.array_dims}")
                    out.append(("heap", arr.tobytes()))
                elif f.kind == FieldKind.VAR_BYTES:
                    out.append(("var", bytes(v)))
                else:
                    codec = config.compress_codec if draw.chance(config.compress_probability) else CodecId.RAW
                    blob = encode_image(np.asarray(v), codec, max_height=f.max_height, max_width=f.max_width,
                                        jpeg=config.jpeg)
                    if blob.channels != f.channels:
                        raise SchemaMismatch(
                            f"sample {i} field {f.name!r}: {blob.channels} channels != {f.channels}")
                    out.append(("image", blob, codec))
            return out

        def encoded():
            if config.num_encode_workers <= 1:
                for i in range(n):
                    yield i, encode_sample(i)
                return
            from concurrent.futures import ThreadPoolExecutor

            chunk = 64 * config.num_encode_workers
            with ThreadPoolExecutor(config.num_encode_workers) as ex:
                for c0 in range(0, n, chunk):
                    for i, enc in zip(range(c0, min(n, c0 + chunk)), ex.map(encode_sample, range(c0, min(n, c0 + chunk)))):
                        yield i, enc

        for i, enc in encoded():   # allocation stays sequential: the layout is worker-count independent
            cells = []
            for item in enc:
                if not isinstance(item, tuple):
                    cells.append(item)
                elif item[0] == "heap":
                    cells.append(heap.put(item[1]))
                elif item[0] == "var":
                    data = item[1]
                    cells.append(VarBytesCell(heap.put(data), len(data)) if data else VarBytesCell(0, 0))
                else:
                    _, blob, codec = item
                    off = heap.put(blob.payload)
                    cells.append(ImageCell(off, len(blob.payload), blob.height, blob.width, blob.channels,
                                           int(codec)))
                    counts[CodecId(codec)] += 1
            rows[i * rw:(i + 1) * rw] = encode_row(schema, cells)
        regions = heap.finish()
        alloc_off = heap_offset + heap.next_page * page
        os.ftruncate(fd, alloc_off)
        os.pwrite(fd, encode_alloc_table(regions), alloc_off)
        os.pwrite(fd, bytes(rows), hlen)
        header = DatasetHeader(n, page, hlen, heap_offset, alloc_off, tuple(schema))
        os.pwrite(fd, encode_header(header), 0)
    except BaseException:
        os.close(fd)
        try:
            os.unlink(path)
        except OSError:
            pass
        raise
    os.close(fd)
    used = sum(r.length for r in regions)
    heap_bytes = heap.next_page * page
    return WriteReport(
        path=str(path), num_samples=n, num_pages=heap.next_page,
        bytes_written=alloc_off + 8 + 16 * len(regions),
        codec_counts={c.name: k for c, k in counts.items() if k},
        waste_fraction=(heap_bytes - used) / heap_bytes if heap_bytes else 0.0,
    )


def read_header(path) -> DatasetHeader:
    from .format import HEADER_PREFIX

    with open(path, "rb") as fh:
        prefix = fh.read(HEADER_PREFIX.size)
        if len(prefix) < HEADER_PREFIX.size:
            raise InvalidFile(f"{path}: file shorter than header prefix")
        nf = HEADER_PREFIX.unpack(prefix)[3]
        fh.seek(0)
        return decode_header(fh.read(header_byte_length(nf)))


def report_waste(path) -> float:
    try:
        h = read_header(path)
    except InvalidFile:
        raise
    except Exception as e:
        raise InvalidFile(f"{path}: {e}") from e
    with open(path, "rb") as fh:
        fh.seek(h.alloc_table_offset)
        regions = decode_alloc_table(fh.read())
    if h.heap_bytes == 0:
        return 0.0
    return (h.heap_bytes - sum(r.length for r in regions)) / h.heap_bytes
