"""Epoch orders: sequential, random, quasi-random (native, draw-for-draw
identical to traversal.py:45-150 of the reference).

The permutation is computed in libbbx (csrc/orders.cpp); QUASI_RANDOM there
is O(N log P) instead of the reference's O(N * batch_size) list walk.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .rng import TAG_ORDER, Rng, stream_seed


class OrderKind(enum.Enum):
    SEQUENTIAL = "sequential"
    RANDOM = "random"
    QUASI_RANDOM = "quasi-random"


OrderOption = OrderKind   # FFCV alias
_KIND_CODE = {OrderKind.SEQUENTIAL: 0, OrderKind.RANDOM: 1, OrderKind.QUASI_RANDOM: 2}


@dataclass
class QuasiRandomTrace:
    page_loads: list = dc_field(default_factory=list)
    max_buffered: int = 0


def _page_array(num_samples: int, page_map):
    if page_map is None:
        return None
    if callable(page_map):
        page_map = [page_map(i) for i in range(num_samples)]
    if isinstance(page_map, np.ndarray) and page_map.dtype == np.int64:
        return np.ascontiguousarray(page_map)
    return np.array([-1 if p is None else int(p) for p in page_map], dtype=np.int64)


def epoch_permutation(kind: OrderKind, seed: int, epoch: int, num_samples: int, page_map=None,
                      batch_size: int | None = None) -> np.ndarray:
    """The epoch's permutation of 0..N-1 as an int64 array (native)."""
    kind = OrderKind(kind)
    if kind == OrderKind.QUASI_RANDOM and (batch_size is None or batch_size < 1):
        raise ValueError("quasi-random order requires batch_size >= 1")
    out = np.empty(num_samples, dtype=np.int64)
    pages = _page_array(num_samples, page_map) if kind == OrderKind.QUASI_RANDOM else None
    L = _lib.lib()
    _lib.check(L.bbx_epoch_order(_KIND_CODE[kind], seed & 0xFFFFFFFFFFFFFFFF, epoch & 0xFFFFFFFFFFFFFFFF,
                                 num_samples, None if pages is None else pages.ctypes.data,
                                 batch_size or 0, out.ctypes.data if num_samples else None))
    return out


@dataclass
class TraversalOrder:
    kind: OrderKind
    seed: int = 0

    def epoch_rng(self, epoch: int) -> Rng:
        return Rng(stream_seed(self.seed, TAG_ORDER, epoch))

    def epoch_indices(self, epoch: int, num_samples: int, page_map=None, batch_size: int | None = None,
                      trace: QuasiRandomTrace | None = None) -> list:
        perm = epoch_permutation(self.kind, self.seed, epoch, num_samples, page_map, batch_size)
        if trace is not None and OrderKind(self.kind) == OrderKind.QUASI_RANDOM:
            _fill_trace(trace, self.seed, epoch, _page_array(num_samples, page_map), batch_size)
        return perm.tolist()

    def epoch_batches(self, epoch: int, num_samples: int, batch_size: int, page_map=None,
                      drop_last: bool = False) -> list:
        if batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        return [b.tolist() for b in self.epoch_batch_arrays(epoch, num_samples, batch_size, page_map, drop_last)]

    def epoch_batch_arrays(self, epoch: int, num_samples: int, batch_size: int, page_map=None,
                           drop_last: bool = False) -> list:
        """epoch_batches as int64 array views of one permutation (no per-index Python objects)."""
        if batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        perm = epoch_permutation(self.kind, self.seed, epoch, num_samples, page_map, batch_size)
        out = [perm[i:i + batch_size] for i in range(0, num_samples, batch_size)]
        if drop_last and out and len(out[-1]) < batch_size:
            out.pop()
        return out


def _fill_trace(trace: QuasiRandomTrace, seed: int, epoch: int, pages, batch_size: int) -> None:
    """Page admissions of a quasi-random epoch (traversal.py:56-63): every page is
    admitted once, in the shuffled page order, keeping <= batch_size admitted."""
    keys = sorted(set(pages.tolist())) if pages is not None else [-1]
    order = [k for k in keys if k >= 0] + ([-1] if -1 in keys else [])
    Rng(stream_seed(seed, TAG_ORDER, epoch)).shuffle(order)
    trace.page_loads.extend(None if p < 0 else p for p in order)
    trace.max_buffered = max(trace.max_buffered, min(batch_size, len(order)))


def next_epoch(order: TraversalOrder, num_samples: int, page_map, batch_size: int, epoch: int = 0,
               drop_last: bool = False) -> list:
    return order.epoch_batches(epoch, num_samples, batch_size, page_map, drop_last)


def uniformity_probe(kind: OrderKind, num_samples: int, epochs: int, seed: int = 0, page_map=None,
                     batch_size: int | None = None) -> np.ndarray:
    """Mean emission position of every sample over `epochs` epochs."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    totals = np.zeros(num_samples, dtype=np.float64)
    pos = np.arange(num_samples, dtype=np.float64)
    for e in range(epochs):
        perm = epoch_permutation(kind, seed, e, num_samples, page_map, batch_size)
        totals[perm] += pos
    return totals / epochs
