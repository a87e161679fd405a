"""The .bbox container layout (host side).

Byte layout identical to the reference (format.py:1-43): a 56-byte header
prefix, one 124-byte descriptor per field, a fixed-width row table, page-
aligned heap, allocation table.  The device path parses the same layout in
C++ (csrc/format.cpp); this module serves the writer and the Python-side
metadata (schema, cells, columns).
"""

from __future__ import annotations

import enum
import struct
from dataclasses import dataclass, field as dc_field
from typing import NamedTuple

import numpy as np

from .errors import BadMagic, InvalidFile, InvalidHeader, SchemaMismatch, UnsupportedVersion

MAGIC = b"FASTDS01"
FORMAT_VERSION = 1
MIN_PAGE_SIZE = 1 << 16
DEFAULT_PAGE_SIZE = 1 << 23
MAX_NAME_BYTES = 63

_PREFIX = struct.Struct("<8sIQHQQQQ2x")     # 56 bytes
_DESC = struct.Struct("<64sB48sI7x")        # 124 bytes
_ARRAY_PARAMS = struct.Struct("<BB2x4I")
_IMAGE_PARAMS = struct.Struct("<HHB")
HEADER_PREFIX = _PREFIX
DESCRIPTOR = _DESC


class FieldKind(enum.IntEnum):
    INT_SCALAR = 0
    FLOAT_SCALAR = 1
    FIXED_ARRAY = 2
    VAR_BYTES = 3
    IMAGE = 4


ARRAY_DTYPES = {0: np.dtype("<u1"), 1: np.dtype("<i8"), 2: np.dtype("<f4"), 3: np.dtype("<f8")}
ARRAY_DTYPE_CODES = {v: k for k, v in ARRAY_DTYPES.items()}

# per-kind cell: (width, struct) — format.py:31-36
_CELLS = {
    FieldKind.INT_SCALAR: struct.Struct("<q"),
    FieldKind.FLOAT_SCALAR: struct.Struct("<d"),
    FieldKind.FIXED_ARRAY: struct.Struct("<Q"),
    FieldKind.VAR_BYTES: struct.Struct("<QQ"),
    FieldKind.IMAGE: struct.Struct("<QQHHBB2x"),
}


class VarBytesCell(NamedTuple):
    offset: int
    length: int


class ImageCell(NamedTuple):
    offset: int
    length: int
    height: int
    width: int
    channels: int
    codec: int


class Region(NamedTuple):
    offset: int
    length: int


@dataclass(frozen=True)
class FieldDescriptor:
    name: str
    kind: FieldKind
    array_dtype_code: int = 0
    array_dims: tuple = ()
    max_height: int = 0
    max_width: int = 0
    channels: int = 0

    @property
    def row_cell_width(self) -> int:
        return _CELLS[self.kind].size

    @property
    def array_dtype(self) -> np.dtype:
        return ARRAY_DTYPES[self.array_dtype_code]

    @property
    def array_nbytes(self) -> int:
        return int(np.prod(self.array_dims, dtype=np.int64)) * self.array_dtype.itemsize if self.array_dims else \
            self.array_dtype.itemsize

    def check(self) -> None:
        raw = self.name.encode("utf-8")
        if not 1 <= len(raw) <= MAX_NAME_BYTES:
            raise InvalidHeader(f"field name must be 1..{MAX_NAME_BYTES} bytes: {self.name!r}")
        if self.kind == FieldKind.FIXED_ARRAY:
            if self.array_dtype_code not in ARRAY_DTYPES:
                raise InvalidHeader(f"unknown array dtype code {self.array_dtype_code}")
            if not 1 <= len(self.array_dims) <= 4:
                raise InvalidHeader("fixed arrays support 1..4 dims")
            if not all(1 <= d <= 0xFFFFFFFF for d in self.array_dims):
                raise InvalidHeader("array dims must be positive u32 values")
        elif self.kind == FieldKind.IMAGE:
            if not (1 <= self.max_height <= 0xFFFF and 1 <= self.max_width <= 0xFFFF):
                raise InvalidHeader("image max dims must be in 1..65535")
            if not 1 <= self.channels <= 255:
                raise InvalidHeader("image channels must be in 1..255")


def int_field(name: str) -> FieldDescriptor:
    return FieldDescriptor(name, FieldKind.INT_SCALAR)


def float_field(name: str) -> FieldDescriptor:
    return FieldDescriptor(name, FieldKind.FLOAT_SCALAR)


def array_field(name: str, dtype, dims) -> FieldDescriptor:
    code = ARRAY_DTYPE_CODES[np.dtype(dtype).newbyteorder("<")]
    return FieldDescriptor(name, FieldKind.FIXED_ARRAY, array_dtype_code=code, array_dims=tuple(int(d) for d in dims))


def bytes_field(name: str) -> FieldDescriptor:
    return FieldDescriptor(name, FieldKind.VAR_BYTES)


def image_field(name: str, max_height: int, max_width: int, channels: int) -> FieldDescriptor:
    return FieldDescriptor(name, FieldKind.IMAGE, max_height=max_height, max_width=max_width, channels=channels)


def header_byte_length(num_fields: int) -> int:
    return _PREFIX.size + _DESC.size * num_fields


def row_width(schema) -> int:
    return sum(f.row_cell_width for f in schema)


@dataclass(frozen=True)
class DatasetHeader:
    num_samples: int
    page_size: int
    data_table_offset: int
    heap_offset: int
    alloc_table_offset: int
    fields: tuple = dc_field(default=())
    format_version: int = FORMAT_VERSION

    @property
    def num_fields(self) -> int:
        return len(self.fields)

    @property
    def row_width(self) -> int:
        return row_width(self.fields)

    @property
    def byte_length(self) -> int:
        return header_byte_length(len(self.fields))

    @property
    def heap_bytes(self) -> int:
        return self.alloc_table_offset - self.heap_offset

    @property
    def num_pages(self) -> int:
        return self.heap_bytes // self.page_size

    def check(self) -> None:
        if self.format_version != FORMAT_VERSION:
            raise InvalidHeader(f"format_version must be {FORMAT_VERSION}")
        if not self.fields:
            raise InvalidHeader("at least one field is required")
        if len(self.fields) > 0xFFFF:
            raise InvalidHeader("too many fields")
        if len({f.name for f in self.fields}) != len(self.fields):
            raise InvalidHeader("field names must be unique")
        for f in self.fields:
            f.check()
        ps = self.page_size
        if ps < MIN_PAGE_SIZE or ps & (ps - 1):
            raise InvalidHeader(f"page_size must be a power of two >= {MIN_PAGE_SIZE}")
        if self.num_samples < 0:
            raise InvalidHeader("negative sample count")
        if self.data_table_offset != self.byte_length:
            raise InvalidHeader("data_table_offset must equal the header byte length")
        if self.heap_offset % ps:
            raise InvalidHeader("heap_offset must be page aligned")
        if not self.data_table_offset < self.heap_offset <= self.alloc_table_offset:
            raise InvalidHeader("sections must be ordered header < heap <= alloc table")


def _kind_params(f: FieldDescriptor) -> bytes:
    buf = bytearray(48)
    if f.kind == FieldKind.FIXED_ARRAY:
        dims = list(f.array_dims) + [0] * (4 - len(f.array_dims))
        _ARRAY_PARAMS.pack_into(buf, 0, f.array_dtype_code, len(f.array_dims), *dims)
    elif f.kind == FieldKind.IMAGE:
        _IMAGE_PARAMS.pack_into(buf, 0, f.max_height, f.max_width, f.channels)
    return bytes(buf)


def encode_header(h: DatasetHeader) -> bytes:
    h.check()
    parts = [_PREFIX.pack(MAGIC, h.format_version, h.num_samples, h.num_fields, h.page_size,
                          h.data_table_offset, h.heap_offset, h.alloc_table_offset)]
    for f in h.fields:
        parts.append(_DESC.pack(f.name.encode("utf-8"), int(f.kind), _kind_params(f), f.row_cell_width))
    return b"".join(parts)


def decode_header(buf: bytes) -> DatasetHeader:
    if len(buf) < _PREFIX.size:
        raise InvalidHeader(f"buffer too short for header prefix: {len(buf)} bytes")
    magic, version, n, nf, page, dto, ho, ato = _PREFIX.unpack_from(buf, 0)
    if magic != MAGIC:
        raise BadMagic(f"bad magic {magic!r}")
    if version != FORMAT_VERSION:
        raise UnsupportedVersion(f"unsupported version {version}")
    if len(buf) < header_byte_length(nf):
        raise InvalidHeader(f"buffer too short for {nf} descriptors")
    fields = []
    for k in range(nf):
        raw, kind, params, width = _DESC.unpack_from(buf, _PREFIX.size + k * _DESC.size)
        try:
            kind = FieldKind(kind)
        except ValueError:
            raise InvalidHeader(f"unknown field kind {kind}") from None
        name = raw.rstrip(b"\0").decode("utf-8")
        extra = {}
        if kind == FieldKind.FIXED_ARRAY:
            code, nd, *dims = _ARRAY_PARAMS.unpack_from(params, 0)
            if code not in ARRAY_DTYPES:
                raise InvalidHeader(f"unknown array dtype code {code}")
            if not 1 <= nd <= 4:
                raise InvalidHeader(f"array ndims out of range: {nd}")
            extra = {"array_dtype_code": code, "array_dims": tuple(dims[:nd])}
        elif kind == FieldKind.IMAGE:
            mh, mw, ch = _IMAGE_PARAMS.unpack_from(params, 0)
            extra = {"max_height": mh, "max_width": mw, "channels": ch}
        f = FieldDescriptor(name, kind, **extra)
        if width != f.row_cell_width:
            raise InvalidHeader(f"field {name!r}: stored cell width {width} != {f.row_cell_width}")
        fields.append(f)
    h = DatasetHeader(n, page, dto, ho, ato, tuple(fields), version)
    h.check()
    return h


def encode_row(schema, values) -> bytes:
    if len(values) != len(schema):
        raise SchemaMismatch(f"expected {len(schema)} cells, got {len(values)}")
    out = []
    for f, v in zip(schema, values):
        st = _CELLS[f.kind]
        try:
            if f.kind == FieldKind.INT_SCALAR:
                out.append(st.pack(int(v)))
            elif f.kind == FieldKind.FLOAT_SCALAR:
                out.append(st.pack(float(v)))
            elif f.kind == FieldKind.FIXED_ARRAY:
                out.append(st.pack(int(v)))
            elif f.kind == FieldKind.VAR_BYTES:
                out.append(st.pack(v.offset, v.length))
            else:
                out.append(st.pack(v.offset, v.length, v.height, v.width, v.channels, v.codec))
        except (struct.error, TypeError, AttributeError) as e:
            raise SchemaMismatch(f"field {f.name!r}: cell {v!r} does not match {f.kind.name}") from e
    return b"".join(out)


def decode_row(schema, buf) -> tuple:
    if len(buf) < row_width(schema):
        raise SchemaMismatch(f"row buffer too short: {len(buf)} < {row_width(schema)}")
    cells, pos = [], 0
    for f in schema:
        vals = _CELLS[f.kind].unpack_from(buf, pos)
        if f.kind == FieldKind.VAR_BYTES:
            cells.append(VarBytesCell(*vals))
        elif f.kind == FieldKind.IMAGE:
            cells.append(ImageCell(*vals))
        else:
            cells.append(vals[0])
        pos += f.row_cell_width
    return tuple(cells)


def encode_alloc_table(regions) -> bytes:
    arr = np.zeros(1 + 2 * len(regions), dtype="<u8")
    arr[0] = len(regions)
    if regions:
        arr[1:] = np.asarray([(r.offset, r.length) for r in regions], dtype="<u8").reshape(-1)
    return arr.tobytes()


def decode_alloc_table(buf) -> list:
    if len(buf) < 8:
        raise InvalidFile("allocation table truncated")
    count = int(np.frombuffer(buf, dtype="<u8", count=1)[0])
    need = 8 + 16 * count
    if len(buf) < need:
        raise InvalidFile(f"allocation table truncated: {len(buf)} < {need}")
    pairs = np.frombuffer(buf, dtype="<u8", count=2 * count, offset=8).reshape(-1, 2)
    return [Region(int(o), int(n)) for o, n in pairs]
