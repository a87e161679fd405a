"""Epoch orchestration on the GPU: order -> device pipeline -> batch leases.

Drop-in for loader.py:37-453 of the reference: same `LoaderConfig`,
`Loader(dataset_or_path, config)`, `iterate_epoch`, `Batch` lease semantics
(valid until the next batch is requested), `EpochStats`, error reporting
("sample {index} failed: {err}" with the reference's exception type).

What replaces the reference's N worker threads x per-sample Python
(_EpochRun._process_position, loader.py:330-347) is one libbbx loader per
Loader: each batch is a single `bbx_loader_submit` (indices in, everything
else on the device), slot_count ring slots of device output tensors, and a
prefetch depth of slot_count - 1 batches.  Batch arrays are CUDA tensors,
channels-last (NHWC), exactly the reference's numpy shapes and dtypes.

Stream semantics (as FFCV's loader): a yielded batch's device work is ordered
before the work queued afterwards on the CUDA stream that was current when the
iteration started (bbx_loader_stream_wait); the host does not wait for it unless
the batch has device-detected sample errors to read (RLE / JPEG fields).  Work on
another stream must wait on that stream (e.g. `other.wait_stream(current)`).

Extensions: `distributed=True` shards every global batch of
world_size * batch_size positions by rank; `device`.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import pipeline as pl
from .errors import CapacityTooSmall, SchemaMismatch, ShutdownError, SpecMismatch
from .format import FieldKind
from .reader import Dataset, DeviceResident, Direct, OsCache, ProcessCacheStrategy, open_dataset
from .traversal import OrderKind, TraversalOrder

DEFAULT_SLOT_COUNT = 3


@dataclass
class LoaderConfig:
    batch_size: int
    num_workers: int = 1
    slot_count: int = DEFAULT_SLOT_COUNT
    order: OrderKind = OrderKind.RANDOM
    seed: int = 0
    drop_last: bool = False
    pipelines: dict | None = None
    fields: list | None = None
    # ---- extensions (no reference counterpart)
    device: int | None = None          # CUDA ordinal; default LOCAL_RANK / current device
    distributed: bool = False          # shard each global batch by rank (FFCV distributed=True)
    rank: int | None = None
    world_size: int | None = None
    staging_threads: int = 0           # host gather threads (0 = automatic)
    options: dict | None = None        # engine tuning options (include/bbx.h bbx_loader_set_option); defaults = measured best

    def check(self) -> None:
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.num_workers < 1:
            raise ValueError("num_workers must be >= 1")
        if self.slot_count < 2:
            raise ValueError("slot_count must be >= 2")


@dataclass
class EpochStats:
    batches: int = 0
    samples: int = 0
    page_fetches: int = 0
    page_reloads: int = 0
    producer_blocked_s: float = 0.0
    consumer_blocked_s: float = 0.0


class Batch:
    """A lease on one ring slot's device tensors; valid until the next batch."""

    __slots__ = ("arrays", "_idx", "_list", "index")

    def __init__(self, arrays: dict, indices, index: int):
        self.arrays = arrays
        self._idx = indices          # list or int64 ndarray; `indices` is a list, as the reference's
        self._list = indices if isinstance(indices, list) else None
        self.index = index

    @property
    def indices(self) -> list:
        """The batch's sample indices (a list, loader.py:411), built on first access."""
        if self._list is None:
            self._list = self._idx.tolist()
        return self._list

    def __getitem__(self, name: str):
        return self.arrays[name]

    def __contains__(self, name) -> bool:
        return name in self.arrays

    @property
    def size(self) -> int:
        return len(self._idx)

    def keys(self):
        return self.arrays.keys()


class MemoryLedger:
    def __init__(self):
        self.entries: dict = {}

    def register(self, name: str, nbytes: int) -> None:
        self.entries[name] = nbytes

    @property
    def total(self) -> int:
        return sum(self.entries.values())


_TORCH_DT = None


def _torch_dtype(code: int):
    global _TORCH_DT
    import torch

    if _TORCH_DT is None:
        _TORCH_DT = {_lib.DT_U8: torch.uint8, _lib.DT_I64: torch.int64, _lib.DT_F32: torch.float32,
                     _lib.DT_F64: torch.float64, _lib.DT_F16: torch.float16, _lib.DT_BF16: torch.bfloat16}
    return _TORCH_DT[code]


def _dist_info(config: LoaderConfig) -> tuple[int, int]:
    if not config.distributed:
        return 0, 1
    rank, world = config.rank, config.world_size
    if rank is None or world is None:
        try:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                rank = dist.get_rank() if rank is None else rank
                world = dist.get_world_size() if world is None else world
        except Exception:
            pass
    rank = int(os.environ.get("RANK", 0)) if rank is None else rank
    world = int(os.environ.get("WORLD_SIZE", 1)) if world is None else world
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return rank, world


def agree_seed(config: LoaderConfig, device: int | None = None) -> int:
    """distributed=True: the one collective of the path -- at construction, every
    rank adopts rank 0's seed (one broadcast), so all ranks compute the same global
    order and per-sample parameters.  No collective runs per batch."""
    if not config.distributed:
        return config.seed
    try:
        import torch
        import torch.distributed as dist
    except Exception:
        return config.seed
    if not (dist.is_available() and dist.is_initialized()):
        return config.seed
    dev = "cpu"
    if dist.get_backend() == "nccl":
        dev = f"cuda:{device if device is not None else torch.cuda.current_device()}"
    u = config.seed & 0xFFFFFFFFFFFFFFFF             # the full 64-bit seed, as two's-complement int64
    t = torch.tensor([u - (1 << 64) if u >= (1 << 63) else u], dtype=torch.int64, device=dev)
    dist.broadcast(t, src=0)
    return int(t.item()) & 0xFFFFFFFFFFFFFFFF


def _fits_pinned(nbytes: int, fraction: float) -> bool:
    try:
        ram = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        return False
    local = int(os.environ.get("LOCAL_WORLD_SIZE", 1))
    return nbytes <= fraction * ram / max(local, 1)


def shard_batches(global_batches: list, rank: int, world_size: int, batch_size: int) -> list:
    """Rank r's share of every global batch of world_size * B positions.

    A full global batch gives rank r positions [r*B, (r+1)*B).  A short tail of
    t positions is padded to t' = ceil(t / W) * W by wrapping around to the
    epoch's first indices (as torch's DistributedSampler pads) and split evenly,
    t' / W positions per rank, so every rank gets the same number of batches and
    a DDP step never waits on a rank that has run out."""
    out = []
    full = world_size * batch_size
    for gb in global_batches:
        gb = np.asarray(gb, dtype=np.int64)
        if len(gb) == full or world_size == 1:
            out.append(gb[rank * batch_size:(rank + 1) * batch_size])
            continue
        t = len(gb)
        per = -(-t // world_size)
        pad = per * world_size - t
        if pad:                                      # pad < W: the epoch's first indices (cycled)
            head, have = [], 0
            for b in global_batches:
                head.append(np.asarray(b, dtype=np.int64))
                have += len(head[-1])
                if have >= pad:
                    break
            first = np.concatenate(head)
            gb = np.concatenate([gb, first[np.arange(pad) % len(first)]])
        out.append(gb[rank * per:(rank + 1) * per])
    return out


class _Field:
    __slots__ = ("name", "plan_id", "outs", "nchw", "scalar", "contiguous", "views")

    def __init__(self, name, plan_id, outs, nchw, scalar, contiguous=False):
        self.name, self.plan_id, self.outs, self.nchw, self.scalar = name, plan_id, outs, nchw, scalar
        # per-slot views made once (indexing a tensor costs microseconds per batch)
        self.views = [outs[k].permute(0, 3, 1, 2) if nchw else outs[k] for k in range(outs.shape[0])]
        self.contiguous = contiguous


class Loader:
    """Batch loader over an open dataset (or a path, which it then owns)."""

    def __init__(self, dataset, config: LoaderConfig):
        import torch

        config.check()
        self._owns_dataset = isinstance(dataset, (str, bytes)) or hasattr(dataset, "__fspath__")
        self.dataset: Dataset = open_dataset(dataset) if self._owns_dataset else dataset
        self.config = config
        self.order = TraversalOrder(config.order, config.seed)
        self.ledger = MemoryLedger()
        self.last_stats: EpochStats | None = None
        self._auto_epoch = 0
        self._shutdown = False
        self._epoch_lock = threading.Lock()
        self._active = None
        self._handle = None
        self._headers_named = False
        self.rank, self.world_size = _dist_info(config)
        if config.device is not None:
            self.device = int(config.device)
        elif config.distributed and "LOCAL_RANK" in os.environ:
            self.device = int(os.environ["LOCAL_RANK"])
        else:
            self.device = torch.cuda.current_device()
        if config.distributed:   # one-time seed agreement (the only cross-rank traffic)
            seed = agree_seed(config, self.device)
            if seed != config.seed & 0xFFFFFFFFFFFFFFFF:
                config = dataclasses.replace(config, seed=seed)
                self.config = config
                self.order = TraversalOrder(config.order, config.seed)

        schema = self.dataset.schema
        wanted = config.fields
        self.batch_fields = []
        for f in schema:
            if wanted is not None and f.name not in wanted:
                continue
            if f.kind == FieldKind.VAR_BYTES:
                if wanted is not None:
                    raise SchemaMismatch(f"field {f.name!r}: VAR_BYTES fields cannot be batched")
                continue
            self.batch_fields.append(f)
        if not self.batch_fields:
            raise SchemaMismatch("no batchable fields selected")

        strategy = self.dataset.strategy
        self.page_pool = isinstance(strategy, ProcessCacheStrategy)
        self.direct_io = isinstance(strategy, Direct)
        if isinstance(strategy, DeviceResident):
            if isinstance(strategy, DeviceResident) and strategy.device is not None and \
                    int(strategy.device) != self.device:
                raise ValueError(f"DeviceResident(device={strategy.device}) but the loader runs on cuda:{self.device}: "
                                 "the kernels read the heap from the loader's own device")
            self.dataset.make_resident(self.device)
        elif isinstance(strategy, OsCache) and strategy.pinned and not self.dataset.pinned:
            if not _fits_pinned(self.dataset.header.heap_bytes, OsCache.PIN_HOST_RAM_FRACTION):
                raise CapacityTooSmall("heap does not fit the pinned host budget")
            self.dataset.pin_host()

        L = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(L.bbx_loader_create(self.dataset.handle, self.device, config.batch_size, config.slot_count,
                                       config.staging_threads, ctypes.byref(h)))
        self._handle = h
        if isinstance(strategy, OsCache) and getattr(strategy, "zero_copy", False):
            _lib.check(L.bbx_loader_set_zero_copy(h, 1))
        if isinstance(strategy, Direct):   # one pread per payload, the strategy's latency first
            _lib.check(L.bbx_loader_set_option(h, b"direct_io", 1))
            _lib.check(L.bbx_loader_set_option(h, b"read_latency_ns", int(strategy.read_latency_s * 1e9)))
        if self.page_pool:   # HBM page pool executing the reference's PageSchedule (reader.py:96-297)
            strategy.check()
            _lib.check(L.bbx_loader_set_page_pool(h, int(strategy.capacity_pages), float(strategy.fetch_latency_s)))
        for name, value in (config.options or {}).items():
            _lib.check(L.bbx_loader_set_option(h, str(name).encode(), int(value)))
        field_index = {f.name: i for i, f in enumerate(schema)}
        self._field_index = field_index
        pipelines = dict(config.pipelines or {})
        self._fields: list[_Field] = []
        self.scalar_fields = []
        B, S = config.batch_size, config.slot_count
        dev = torch.device("cuda", self.device)
        try:
            for f in self.batch_fields:
                fi = field_index[f.name]
                if f.kind in (FieldKind.INT_SCALAR, FieldKind.FLOAT_SCALAR):
                    if f.name in pipelines:
                        raise SchemaMismatch(f"scalar field {f.name!r} cannot take a pipeline")
                    pid = ctypes.c_int32()
                    _lib.check(L.bbx_loader_add_scalar(h, fi, ctypes.byref(pid)))
                    dt = torch.int64 if f.kind == FieldKind.INT_SCALAR else torch.float64
                    outs = torch.empty((S, B), dtype=dt, device=dev)
                    self.scalar_fields.append(f)
                    self._fields.append(_Field(f.name, pid.value, outs, False, True))
                    self.ledger.register(f"scalars:{f.name}", outs.numel() * outs.element_size())
                    continue
                chain = pipelines.pop(f.name, None) or pl.default_chain_for_field(f)
                if not isinstance(chain[0], pl.SourceTransform):
                    chain = pl.default_chain_for_field(f)[:1] + list(chain)
                comp = pl.compile_chain(chain, pl.input_spec_for_field(f))
                ops = (_lib.BbxOp * len(comp.ops))(*comp.ops)
                pid, nd, odt = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
                shape = (ctypes.c_int64 * 4)()
                _lib.check(L.bbx_loader_add_field(h, fi, ops, len(comp.ops), ctypes.byref(pid), shape,
                                                  ctypes.byref(nd), ctypes.byref(odt)))
                oshape = tuple(int(shape[k]) for k in range(nd.value))
                want_shape = tuple(comp.specs[-1][0])
                if oshape != want_shape:
                    raise SpecMismatch(f"device plan shape {oshape} != spec {want_shape}")
                outs = torch.empty((S, B, *oshape), dtype=_torch_dtype(odt.value), device=dev)
                self._fields.append(_Field(f.name, pid.value, outs, comp.nchw_view, False, comp.nchw_contiguous))
                self.ledger.register(f"arena:{f.name}", outs.numel() * outs.element_size())
            if pipelines:
                raise SchemaMismatch(f"pipelines for unknown fields: {sorted(pipelines)}")
            for fd in self._fields:
                for s in range(S):
                    _lib.check(L.bbx_loader_bind(h, fd.plan_id, s, fd.outs[s].data_ptr()))
        except BaseException:
            L.bbx_loader_destroy(h)
            self._handle = None
            if self._owns_dataset:
                self.dataset.close()
            raise
        self.ledger.register("dataset_buffers", self.dataset.tracked_bytes)

    # -- public surface ---------------------------------------------------
    @property
    def tracked_buffer_bytes(self) -> int:
        return self.ledger.total

    @property
    def handle(self):
        return self._handle

    def batches_per_epoch(self) -> int:
        """The same on every rank (a short tail global batch is padded, shard_batches)."""
        n = self.dataset.num_samples
        gb = self.config.batch_size * self.world_size
        return n // gb if self.config.drop_last else -(-n // gb)

    def epoch_batches(self, epoch: int) -> list:
        """This rank's index lists for `epoch` (the reference order, then sharded)."""
        return [b.tolist() for b in self._epoch_batch_arrays(epoch)]

    def _epoch_batch_arrays(self, epoch: int) -> list:
        cfg = self.config
        page_map = self.dataset.page_map() if OrderKind(cfg.order) == OrderKind.QUASI_RANDOM else None
        gbs = cfg.batch_size * self.world_size
        batches = self.order.epoch_batch_arrays(epoch, self.dataset.num_samples, gbs, page_map, cfg.drop_last)
        if self.world_size > 1:
            batches = shard_batches(batches, self.rank, self.world_size, cfg.batch_size)
        return batches

    def iterate_epoch(self, epoch: int = 0):
        if self._shutdown:
            raise ShutdownError("loader is shut down")
        run = _EpochRun(self, epoch)
        with self._epoch_lock:
            self._active = run
        try:
            yield from run.batches()
        finally:
            run.stop()
            self.last_stats = run.stats
            with self._epoch_lock:
                self._active = None

    def iterate_steps(self, steps: int, start_epoch: int = 0):
        """`steps` batches as one continuous stream over epochs start_epoch,
        start_epoch+1, ... (each batch identical to the same batch of
        iterate_epoch); the prefetch pipeline is not drained at epoch ends."""
        if self._shutdown:
            raise ShutdownError("loader is shut down")
        run = _EpochRun(self, start_epoch, steps)
        with self._epoch_lock:
            self._active = run
        try:
            yield from run.batches()
        finally:
            run.stop()
            self.last_stats = run.stats
            with self._epoch_lock:
                self._active = None

    def set_profiling(self, enabled: bool | int = True) -> None:
        """CUDA-event timing of the transform kernels (stats()['kernel_seconds']);
        an int n > 1 times every n-th batch only (the events' cost stays off the rest)."""
        _lib.check(_lib.lib().bbx_loader_set_profiling(self._handle, int(enabled)))

    def reset_stats(self) -> None:
        _lib.check(_lib.lib().bbx_loader_reset_stats(self._handle))

    def __iter__(self):
        epoch = self._auto_epoch
        self._auto_epoch += 1
        return self.iterate_epoch(epoch)

    def __len__(self) -> int:
        return self.batches_per_epoch()

    def stats(self) -> dict:
        st = _lib.LoaderStats()
        _lib.check(_lib.lib().bbx_loader_get_stats(self._handle, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in st._fields_}

    def shutdown(self) -> None:
        if self._shutdown:
            return
        self._shutdown = True
        with self._epoch_lock:
            run = self._active
        if run is not None:
            run.stop()
        if self._handle is not None:
            _lib.lib().bbx_loader_destroy(self._handle)
            self._handle = None
        if self._owns_dataset:
            self.dataset.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()

    def __del__(self):
        try:
            self.shutdown()
        except Exception:
            pass


class _EpochRun:
    """One epoch: submit ahead by slot_count - 1 batches, lease one at a time."""

    def __init__(self, loader: Loader, epoch: int, steps: int | None = None):
        self.loader = loader
        self.epoch = epoch
        self.stats = EpochStats()
        # batch index arrays, extended an epoch at a time as the stream needs them
        # (iterate_steps: a continuous stream across epoch boundaries, no pipeline drain)
        self.batch_lists, self.batch_epochs = [], []
        self._steps = steps
        self._next_epoch = epoch
        self._exhausted = False
        self._ensure(0)
        if steps is None:
            self._exhausted = True                      # exactly one epoch
        self._inflight: set = set()
        self._stopped = False

    def _ensure(self, g: int) -> bool:
        """Batch g is known (extending the stream by whole epochs); False past the end."""
        while len(self.batch_lists) <= g and not self._exhausted:
            bl = self.loader._epoch_batch_arrays(self._next_epoch)
            if not bl:
                self._exhausted = True
                break
            if self._steps is not None:
                bl = bl[:self._steps - len(self.batch_lists)]
            if self.loader.page_pool:
                self._plan_pages(bl)
            self.batch_lists += bl
            self.batch_epochs += [self._next_epoch] * len(bl)
            self._next_epoch += 1
            if self._steps is not None and len(self.batch_lists) >= self._steps:
                self._exhausted = True
        return g < len(self.batch_lists)

    def _plan_pages(self, batches) -> None:
        """The epoch's page plan (loader.py:273-291): trace, CapacityTooSmall check
        and the Belady schedule, computed natively and queued ahead of the epoch's
        batches (bbx_loader_plan_epoch)."""
        idx = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.int64) for b in batches])
                                   if batches else np.zeros(0, dtype=np.int64))
        lens = np.ascontiguousarray(np.array([len(b) for b in batches], dtype=np.int32))
        fetches, reloads = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().bbx_loader_plan_epoch(self.loader.handle, idx.ctypes.data, lens.ctypes.data, len(batches),
                                                    ctypes.byref(fetches), ctypes.byref(reloads)))

    def _submit(self, g: int) -> None:
        ld = self.loader
        slot = g % ld.config.slot_count
        idx = np.ascontiguousarray(self.batch_lists[g], dtype=np.int64)
        _lib.check(_lib.lib().bbx_loader_submit(ld.handle, slot, idx.ctypes.data if len(idx) else None, len(idx),
                                                ld.config.seed & 0xFFFFFFFFFFFFFFFF,
                                                self.batch_epochs[g] & 0xFFFFFFFFFFFFFFFF))
        self._inflight.add(slot)

    def batches(self):
        import torch

        ld = self.loader
        L = _lib.lib()
        S = ld.config.slot_count
        if not self._ensure(0):
            return
        stream = torch.cuda.current_stream(ld.device)
        sp = ctypes.c_void_p(stream.cuda_stream)
        if ld.world_size > 1 and not ld._headers_named:
            # before the first submit: this rank's shard of the first epoch is what the
            # loader parses up front (JPEG headers), not every sample of the dataset
            ld._headers_named = True
            mine = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.int64) for b in self.batch_lists]))
            _lib.check(L.bbx_loader_prefetch_headers(ld.handle, mine.ctypes.data, len(mine)))
        pool_base = ld.stats() if ld.page_pool else None   # page-pool counters at the stream's start
        io_seen = ld.stats()["io_reads"] if ld.direct_io else 0
        for g in range(S - 1):
            if self._ensure(g):
                self._submit(g)
        g = 0
        bad = ctypes.c_int64(-1)
        bad_ref = ctypes.byref(bad)
        seed = ld.config.seed & 0xFFFFFFFFFFFFFFFF
        step = L.bbx_loader_step
        while self._ensure(g):
            if self._stopped:
                raise ShutdownError("epoch stopped")
            slot = g % S
            # release the previous lease, submit batch g + S - 1, wait for batch g and
            # order the consumer's stream after it: one call (bbx_loader_step)
            rel, sub, nidx, ep, iptr = -1, -1, 0, 0, None
            if self._ensure(g + S - 1):
                rel = (g - 1) % S if g >= 1 else -1
                sub = (g + S - 1) % S
                sidx = np.ascontiguousarray(self.batch_lists[g + S - 1], dtype=np.int64)
                nidx, ep = len(sidx), self.batch_epochs[g + S - 1] & 0xFFFFFFFFFFFFFFFF
                iptr = sidx.ctypes.data if nidx else None
                self._inflight.add(sub)
            t0 = time.perf_counter()
            rc = step(ld.handle, rel, sub, iptr, nidx, seed, ep, slot, sp, bad_ref)
            self.stats.consumer_blocked_s += time.perf_counter() - t0
            self._inflight.discard(slot)
            indices = self.batch_lists[g]
            if rc != 0:
                exc = _lib.STATUS_EXC.get(rc, Exception)
                msg = _lib.last_error()
                if bad.value >= 0:
                    raise exc(f"sample {int(indices[bad.value])} failed: {msg}")
                raise exc(msg)
            count = len(indices)
            arrays = {}
            full = count == ld.config.batch_size
            for fd in ld._fields:
                t = fd.views[slot]                       # full batches hand out the slot tensor itself
                if not full:
                    t = t[:count]
                if fd.contiguous:                        # ToTorchImage(channels_last=False)
                    t = t.contiguous()
                arrays[fd.name] = t
            self.stats.batches += 1
            self.stats.samples += count
            if ld.direct_io:            # Direct: the loader's preads count as the dataset's reads
                io_now = ld.stats()["io_reads"]
                ld.dataset.io_read_count += io_now - io_seen
                io_seen = io_now
            if pool_base is not None:   # the executed fetches (loader.py:443-445)
                now = ld.stats()
                self.stats.page_fetches = max(0, now["page_fetches"] - pool_base["page_fetches"])
                self.stats.page_reloads = max(0, now["page_reloads"] - pool_base["page_reloads"])
            yield Batch(arrays, indices, g)   # the list is built only if the consumer reads it
            g += 1

    def stop(self) -> None:
        if self._stopped:
            return
        self._stopped = True
        ld = self.loader
        if ld.handle is not None:
            L = _lib.lib()
            L.bbx_loader_drain(ld.handle)   # in-flight batches finish; the ring is reusable
            import torch

            sp = ctypes.c_void_p(torch.cuda.current_stream(ld.device).cuda_stream)
            for s in range(ld.config.slot_count):
                L.bbx_loader_release(ld.handle, s, sp)


def iterate_epoch(dataset, config: LoaderConfig, epoch: int = 0):
    loader = Loader(dataset, config)
    return loader.iterate_epoch(epoch), loader
