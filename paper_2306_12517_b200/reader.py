"""Opening a .bbox container (reader.py:56-546 of the reference, read side).

`Dataset` owns a libbbx dataset handle (mmap + header, csrc/format.cpp) that
the device loader stages payloads from, plus a Python mmap for metadata
(rows, scalar columns, random-access reads).  Strategies:

* OsCache(pinned=None)         page-cache mmap (default; reference OsCache);
                               small heaps are also held pinned for DMA
* Direct(read_latency_s)       every heap read is one pread (+ the latency
                               spun first), counted in io_read_count, as
                               reader.py:61-65,368-372; the loader stages each
                               payload with one pread (loader option direct_io)
* ProcessCacheStrategy(cap)    an HBM page pool of `cap` heap pages executing
                               the reference's Belady PageSchedule per epoch
                               (reader.py:96-297; csrc/engine.cpp page pool):
                               page_fetches / page_reloads as the reference's,
                               CapacityTooSmall as in loader.py:286-289
* DeviceResident(device=None)  extension: the heap lives in HBM (B200 180 GB),
                               batches read payloads from HBM, no H2D per epoch
"""

from __future__ import annotations

import ctypes
import mmap
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .codecs import CodecId, ImageBlob, decode_image
from .errors import CapacityTooSmall, IndexOutOfRange, InvalidFile
from .format import DatasetHeader, FieldKind, decode_row
from .writer import read_header


class OsCache:
    """mmap the file; the OS page cache serves repeated reads.

    pinned: hold the heap page-locked in host RAM so the copy engine DMAs each
    batch's payloads directly (one batched 2-D copy call, no CPU gather).
    Measured on B200 (profiles/): the pooled CPU gather + one contiguous H2D
    is faster for windowed RAW batches (460k vs 163k img/s), so the default
    (None/False) gathers; True opts in (e.g. when host cores are scarce).

    zero_copy: with pinned=True, kernels read each sample's payload window
    straight from the pinned host heap over PCIe (no CPU gather, no staging
    copy).  RAW / SUBSAMPLE2 / array fields only; RLE / JPEG fields stage.
    """

    PIN_HOST_RAM_FRACTION = 0.2

    def __init__(self, pinned: bool | None = None, zero_copy: bool = False):
        self.pinned = pinned or zero_copy
        self.zero_copy = zero_copy


@dataclass
class Direct:
    read_latency_s: float = 0.0


@dataclass
class ProcessCacheStrategy:
    capacity_pages: int
    prefetch_window: int = 8
    fetch_latency_s: float = 0.0

    def check(self) -> None:
        if self.capacity_pages < 1:
            raise CapacityTooSmall(f"capacity_pages must be >= 1, got {self.capacity_pages}")
        if self.prefetch_window < 1:
            raise ValueError("prefetch_window must be >= 1")


@dataclass
class DeviceResident:
    device: int | None = None


class Dataset:
    """An open container; rows are O(1) addressable, payloads staged by libbbx."""

    def __init__(self, path, strategy=None):
        self.path = str(path)
        self.strategy = strategy if strategy is not None else OsCache()
        if isinstance(self.strategy, ProcessCacheStrategy):
            self.strategy.check()
        elif not isinstance(self.strategy, (OsCache, Direct, DeviceResident)):
            raise TypeError(f"unknown read strategy {self.strategy!r}")
        self.header: DatasetHeader = read_header(self.path)
        self.schema = list(self.header.fields)
        self.num_samples = self.header.num_samples
        self.num_pages = self.header.num_pages
        self._row_width = self.header.row_width
        self.io_read_count = 1 if isinstance(self.strategy, Direct) else 0   # the row table (reader.py:343-346)
        self.cache = None
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib().bbx_dataset_open(self.path.encode(), ctypes.byref(handle)), f"{self.path}: ")
        self._handle = handle
        with open(self.path, "rb") as fh:
            self._mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
        self._view = np.frombuffer(self._mm, dtype=np.uint8)
        dto = self.header.data_table_offset
        self._rows = self._view[dto:dto + self.num_samples * self._row_width]
        self._page_map = None
        self._resident_device = None
        self.tracked_bytes = len(self._rows)

    # -- native handle -------------------------------------------------------
    @property
    def handle(self) -> ctypes.c_void_p:
        if self._handle is None:
            raise InvalidFile(f"{self.path}: dataset is closed")
        return self._handle

    def make_resident(self, device: int) -> None:
        """Upload the whole heap to HBM of `device` once (DeviceResident)."""
        if self._resident_device is not None:
            if self._resident_device != device:
                raise ValueError(f"heap already resident on cuda:{self._resident_device}")
            return
        _lib.check(_lib.lib().bbx_dataset_make_resident(self.handle, device))
        self._resident_device = device
        self.tracked_bytes = len(self._rows) + self.header.heap_bytes

    def pin_host(self) -> None:
        """Hold the heap page-locked in host RAM (DMA source for staged batches)."""
        if getattr(self, "_pinned", False):
            return
        _lib.check(_lib.lib().bbx_dataset_pin_host(self.handle, 0))
        self._pinned = True
        self.tracked_bytes += self.header.heap_bytes

    @property
    def pinned(self) -> bool:
        return getattr(self, "_pinned", False)

    @property
    def resident_device(self):
        return self._resident_device

    # -- rows ------------------------------------------------------------------
    def row_bytes(self, i: int) -> bytes:
        if not 0 <= i < self.num_samples:
            raise IndexOutOfRange(f"sample {i} out of range [0, {self.num_samples})")
        w = self._row_width
        return self._rows[i * w:(i + 1) * w].tobytes()

    def cells(self, i: int) -> tuple:
        return decode_row(self.schema, self.row_bytes(i))

    def column(self, name: str) -> np.ndarray:
        off = 0
        for f in self.schema:
            if f.name == name:
                if f.kind not in (FieldKind.INT_SCALAR, FieldKind.FLOAT_SCALAR):
                    raise ValueError(f"column() only reads scalar fields, {name!r} is {f.kind.name}")
                dt = np.dtype("<i8") if f.kind == FieldKind.INT_SCALAR else np.dtype("<f8")
                if self.num_samples == 0:
                    return np.empty(0, dtype=dt)
                table = self._rows.reshape(self.num_samples, self._row_width)
                return np.ascontiguousarray(table[:, off:off + 8]).view(dt).reshape(-1)
            off += f.row_cell_width
        raise KeyError(name)

    # -- pages / heap -----------------------------------------------------------
    def page_of(self, offset: int) -> int:
        return (offset - self.header.heap_offset) // self.header.page_size

    def pages_of_region(self, offset: int, length: int) -> range:
        return range(self.page_of(offset), self.page_of(offset + length - 1) + 1)

    def sample_pages(self, i: int) -> list:
        pages: set = set()
        for f, cell in zip(self.schema, self.cells(i)):
            if f.kind == FieldKind.FIXED_ARRAY:
                pages.update(self.pages_of_region(cell, f.array_nbytes))
            elif f.kind in (FieldKind.VAR_BYTES, FieldKind.IMAGE) and cell.length:
                pages.update(self.pages_of_region(cell.offset, cell.length))
        return sorted(pages)

    def primary_page(self, i: int):
        p = int(self.page_map()[i])
        return None if p < 0 else p

    def page_map(self) -> np.ndarray:
        """Primary page of every sample (-1 = all-inline), computed natively once."""
        if self._page_map is None:
            pm = np.empty(self.num_samples, dtype=np.int64)
            if self.num_samples:
                _lib.check(_lib.lib().bbx_dataset_page_map(self.handle, pm.ctypes.data))
            self._page_map = pm
        return self._page_map

    def heap_read(self, offset: int, length: int, blocking: bool = False) -> np.ndarray:
        if length == 0:
            return np.empty(0, dtype=np.uint8)
        if isinstance(self.strategy, Direct):   # reader.py:368-372: pread copy, latency first
            if self.strategy.read_latency_s:
                end = time.perf_counter() + self.strategy.read_latency_s
                while time.perf_counter() < end:
                    pass
            self.io_read_count += 1
            with open(self.path, "rb", buffering=0) as fh:
                return np.frombuffer(os.pread(fh.fileno(), length, offset), dtype=np.uint8)
        return self._view[offset:offset + length]

    # -- random access ------------------------------------------------------------
    def get_sample(self, i: int, out: dict | None = None) -> dict:
        """Every field of sample i; images are decoded on the GPU (codecs.decode_image)."""
        result = {}
        for f, cell in zip(self.schema, self.cells(i)):
            if f.kind in (FieldKind.INT_SCALAR, FieldKind.FLOAT_SCALAR):
                result[f.name] = cell
            elif f.kind == FieldKind.FIXED_ARRAY:
                raw = self.heap_read(cell, f.array_nbytes)
                result[f.name] = raw.view(f.array_dtype).reshape(f.array_dims).copy()
            elif f.kind == FieldKind.VAR_BYTES:
                result[f.name] = self.heap_read(cell.offset, cell.length).tobytes()
            else:
                blob = ImageBlob(cell.height, cell.width, cell.channels, CodecId(cell.codec),
                                 self.heap_read(cell.offset, cell.length).tobytes())
                target = out.get(f.name) if out else None
                if target is None:
                    target = np.empty((cell.height, cell.width, cell.channels), dtype=np.uint8)
                decode_image(blob, target)
                result[f.name] = target
        return result

    def close(self) -> None:
        if self._handle is not None:
            _lib.lib().bbx_dataset_close(self._handle)
            self._handle = None
        if self._mm is not None:
            self._view = None
            self._rows = None
            try:
                self._mm.close()
            except BufferError:
                pass   # zero-copy views still outstanding
            self._mm = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def open_dataset(path, strategy=None) -> Dataset:
    """Open a container (reader.py:535-546 error wrapping)."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    try:
        return Dataset(path, strategy)
    except (CapacityTooSmall, TypeError, InvalidFile):
        raise
    except Exception as e:
        raise InvalidFile(f"{path}: {e}") from e
