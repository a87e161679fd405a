"""The ctypes module a `bbox` maintainer adds to put the B200 path behind the
reference's own API: `GpuLoader` takes the reference's
`LoaderConfig` and its `Decode` / `RandomCrop` / `RandomFlip` / `Resize` /
`Normalize` / `ToFloat` instances (pipeline.py:95-231), lowers them to bbx_op,
and drives include/bbx.h.  tests/test_gpu_integration.py runs it with the
UNMODIFIED reference package (baseline/_ref) against the reference's goldens."""

import ctypes
from pathlib import Path

import numpy as np
import torch
from bbox import errors as E
from bbox.loader import Batch, LoaderConfig
from bbox.pipeline import Decode, Normalize, RandomCrop, RandomFlip, Resize, ToFloat

_L = ctypes.CDLL(str(Path(__file__).resolve().parents[1] / "paper_2306_12517_b200" / "libbbx.so"))
_EXC = {1: E.InvalidFile, 2: E.BadMagic, 3: E.UnsupportedVersion, 4: E.SchemaMismatch,
        5: E.SpecMismatch, 6: E.CorruptPayload, 7: E.IndexOutOfRange, 8: E.CapacityTooSmall,
        9: E.ShutdownError, 11: E.InvalidHeader, 12: ValueError}


class Op(ctypes.Structure):          # bbx_op
    _fields_ = [("kind", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("p", ctypes.c_double), ("scale", ctypes.c_double * 2),
                ("ratio", ctypes.c_double * 2), ("mean", ctypes.c_float * 4), ("std", ctypes.c_float * 4)]


_vp, _i32, _i64, _u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
for _name, _res, _args in [
        ("bbx_dataset_open", _i32, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
        ("bbx_dataset_close", None, [_vp]),
        ("bbx_loader_create", _i32, [_vp, ctypes.c_int, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
        ("bbx_loader_destroy", None, [_vp]),
        ("bbx_loader_add_field", _i32, [_vp, _i32, ctypes.POINTER(Op), _i32, ctypes.POINTER(_i32),
                                        ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
        ("bbx_loader_add_scalar", _i32, [_vp, _i32, ctypes.POINTER(_i32)]),
        ("bbx_loader_bind", _i32, [_vp, _i32, _i32, _vp]),
        ("bbx_loader_submit", _i32, [_vp, _i32, _vp, _i32, _u64, _u64]),
        ("bbx_loader_wait", _i32, [_vp, _i32, ctypes.POINTER(_i64)]),
        ("bbx_loader_stream_wait", _i32, [_vp, _i32, _vp]),
        ("bbx_loader_release", _i32, [_vp, _i32, _vp]),
        ("bbx_loader_drain", _i32, [_vp]),
        ("bbx_last_error", ctypes.c_char_p, [])]:
    _fn = getattr(_L, _name)
    _fn.restype, _fn.argtypes = _res, _args


def _check(rc):
    if rc:
        raise _EXC.get(rc, E.BboxError)(_L.bbx_last_error().decode())


def _lower(t):                        # Transform instance -> bbx_op (pipeline.py classes)
    o = Op()
    if isinstance(t, Decode):
        o.kind = 0
    elif isinstance(t, ToFloat):
        o.kind = 2
    elif isinstance(t, Normalize):
        o.kind, o.mean[0], o.std[0] = 3, float(t.mean32), float(t.std32)
    elif isinstance(t, RandomFlip):
        o.kind, o.p = 4, t.p
    elif isinstance(t, RandomCrop):
        o.kind, o.h, o.w = 5, t.h, t.w
    elif isinstance(t, Resize):
        o.kind, o.h, o.w = 6, t.h, t.w
    else:
        raise E.SpecMismatch(f"{t!r} has no device lowering")
    return o


class GpuLoader:
    def __init__(self, path, cfg: LoaderConfig, field=0, label=1, device=0):
        self.cfg, ds, ld = cfg, _vp(), _vp()
        _check(_L.bbx_dataset_open(str(path).encode(), ctypes.byref(ds)))
        _check(_L.bbx_loader_create(ds, device, cfg.batch_size, cfg.slot_count, 0, ctypes.byref(ld)))
        self.ds, self.ld = ds, ld
        chain = list((cfg.pipelines or {}).get("image") or [])
        if not chain or not isinstance(chain[0], Decode):
            chain = [Decode()] + chain                  # loader.py:176-178 default source
        ops = (Op * len(chain))(*map(_lower, chain))
        pid, nd, dt, shape = _i32(), _i32(), _i32(), (_i64 * 4)()
        _check(_L.bbx_loader_add_field(ld, field, ops, len(chain), ctypes.byref(pid), shape,
                                       ctypes.byref(nd), ctypes.byref(dt)))
        lid = _i32()
        _check(_L.bbx_loader_add_scalar(ld, label, ctypes.byref(lid)))
        dtype = {0: torch.uint8, 2: torch.float32}[dt.value]
        self.img = torch.empty((cfg.slot_count, cfg.batch_size, *shape[:nd.value]), dtype=dtype, device=device)
        self.lab = torch.empty((cfg.slot_count, cfg.batch_size), dtype=torch.int64, device=device)
        for s in range(cfg.slot_count):
            _check(_L.bbx_loader_bind(ld, pid, s, _vp(self.img[s].data_ptr())))
            _check(_L.bbx_loader_bind(ld, lid, s, _vp(self.lab[s].data_ptr())))

    def iterate_epoch(self, batches, epoch=0):    # batches = TraversalOrder(...).epoch_batches(...)
        S, st = self.cfg.slot_count, _vp(torch.cuda.current_stream().cuda_stream)

        def submit(g):
            idx = np.ascontiguousarray(batches[g], dtype=np.int64)
            _check(_L.bbx_loader_submit(self.ld, g % S, idx.ctypes.data, len(idx), self.cfg.seed, epoch))

        for g in range(min(S - 1, len(batches))):
            submit(g)
        for g in range(len(batches)):
            if g + S - 1 < len(batches):
                if g:
                    _L.bbx_loader_release(self.ld, (g - 1) % S, st)
                submit(g + S - 1)
            bad = _i64()
            rc = _L.bbx_loader_wait(self.ld, g % S, ctypes.byref(bad))
            if rc:
                raise _EXC[rc](f"sample {batches[g][bad.value]} failed: {_L.bbx_last_error().decode()}")
            _check(_L.bbx_loader_stream_wait(self.ld, g % S, st))
            n = len(batches[g])
            yield Batch({"image": self.img[g % S][:n], "label": self.lab[g % S][:n]}, list(batches[g]), g)
        _L.bbx_loader_drain(self.ld)

    def close(self):
        if self.ld:
            _L.bbx_loader_drain(self.ld)
            _L.bbx_loader_destroy(self.ld)
            _L.bbx_dataset_close(self.ds)
            self.ld = self.ds = None
