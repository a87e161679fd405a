"""Transform plugin API, compiled to device op lists.

Same classes, constructor arguments, spec rules and error texts as the
reference's pipeline.py:69-289 (Transform, SourceTransform, Decode,
ArrayRead, ToFloat, Normalize, RandomFlip, RandomCrop, Resize, Opaque,
REGISTRY / parse_pipeline), so a `LoaderConfig.pipelines` written for the
reference builds here unchanged.  What changes is execution: a chain is not
run per sample on the CPU; `compile_chain` lowers it to `bbx_op` records that
libbbx fuses into one sm_100a kernel per field (csrc/kernels.cu: K1).

Extensions (FFCV names; no reference counterpart, parity pinned by our own
oracle): RandomResizedCrop / CenterCrop decoders (bilinear), per-channel
NormalizeImage with float16/bfloat16 output, ToTorchImage (NCHW view).

There is deliberately no CPU `apply`: Opaque stages (arbitrary host
callables, pipeline.py:234-250) cannot run on the device path and are
rejected with SpecMismatch at plan time.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .errors import SpecMismatch
from .format import FieldDescriptor, FieldKind


class Category(enum.Enum):
    FUSIBLE = "fusible"
    OPAQUE = "opaque"


@dataclass(frozen=True)
class ImageSourceSpec:
    max_height: int
    max_width: int
    channels: int


@dataclass(frozen=True)
class ArraySourceSpec:
    shape: tuple
    dtype: np.dtype


def _array_spec(input_spec, who: str):
    if isinstance(input_spec, (ImageSourceSpec, ArraySourceSpec)):
        raise SpecMismatch(f"{who} cannot be first in a chain; start with a source transform")
    shape, dtype = input_spec
    return tuple(shape), np.dtype(dtype)


def _op(kind, **kw) -> L.BbxOp:
    o = L.BbxOp()
    o.kind = kind
    for k, v in kw.items():
        if k in ("mean", "std", "scale", "ratio"):
            arr = getattr(o, k)
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(o, k, v)
    return o


class Transform:
    name = "transform"
    category = Category.FUSIBLE

    def output_spec(self, input_spec):
        raise NotImplementedError

    def prepare(self, input_spec, output_spec) -> None:
        """Plan-time hook (kept for API compatibility; device plans need none)."""

    def to_ops(self, input_spec) -> list:
        raise SpecMismatch(f"transform {self.name!r} has no device lowering")

    def apply(self, inp, out, rng) -> None:
        raise SpecMismatch(f"{type(self).__name__} runs on the device; use it through Loader")

    def __repr__(self) -> str:
        return f"<{type(self).__name__} {self.name}>"


class SourceTransform(Transform):
    def apply_source(self, ref, out, rng) -> None:
        raise SpecMismatch(f"{type(self).__name__} runs on the device; use it through Loader")


class Decode(SourceTransform):
    """Codec dispatch + zero padding to the field's max dims (pipeline.py:95-115)."""

    name = "decode"

    def output_spec(self, input_spec):
        if not isinstance(input_spec, ImageSourceSpec):
            raise SpecMismatch(f"decode expects an image field, got {input_spec!r}")
        return (input_spec.max_height, input_spec.max_width, input_spec.channels), np.dtype(np.uint8)

    def to_ops(self, input_spec):
        return [_op(L.OP_DECODE)]


class ArrayRead(SourceTransform):
    name = "array-read"

    def output_spec(self, input_spec):
        if not isinstance(input_spec, ArraySourceSpec):
            raise SpecMismatch(f"array-read expects an array field, got {input_spec!r}")
        return tuple(input_spec.shape), np.dtype(input_spec.dtype)

    def to_ops(self, input_spec):
        return [_op(L.OP_ARRAYREAD)]


class ToFloat(Transform):
    name = "float"

    def output_spec(self, input_spec):
        shape, _ = _array_spec(input_spec, self.name)
        return shape, np.dtype(np.float32)

    def to_ops(self, input_spec):
        return [_op(L.OP_TOFLOAT)]


class Normalize(Transform):
    """(x - mean) / std in strict float32: one subtract, one divide (pipeline.py:143-160)."""

    name = "normalize"

    def __init__(self, mean: float, std: float):
        if std == 0:
            raise SpecMismatch("normalize std must be nonzero")
        self.mean32 = np.float32(mean)
        self.std32 = np.float32(std)

    def output_spec(self, input_spec):
        shape, _ = _array_spec(input_spec, self.name)
        return shape, np.dtype(np.float32)

    def to_ops(self, input_spec):
        return [_op(L.OP_NORMALIZE, mean=[float(self.mean32)], std=[float(self.std32)])]


class RandomFlip(Transform):
    """Horizontal flip with probability p; one chance() draw (none for p in {0, 1})."""

    name = "flip"

    def __init__(self, p: float = 0.5):
        self.p = p

    def output_spec(self, input_spec):
        shape, dtype = _array_spec(input_spec, self.name)
        if len(shape) != 3:
            raise SpecMismatch("flip expects HxWxC input")
        return shape, dtype

    def to_ops(self, input_spec):
        return [_op(L.OP_FLIP, p=float(self.p))]


class RandomCrop(Transform):
    """Uniform crop over the (padded) input; draws top then left."""

    name = "crop"

    def __init__(self, height: int, width: int):
        self.h = height
        self.w = width

    def output_spec(self, input_spec):
        shape, dtype = _array_spec(input_spec, self.name)
        if len(shape) != 3 or shape[0] < self.h or shape[1] < self.w:
            raise SpecMismatch(f"cannot crop {shape} to {self.h}x{self.w}")
        return (self.h, self.w, shape[2]), dtype

    def to_ops(self, input_spec):
        return [_op(L.OP_CROP, h=self.h, w=self.w)]


class Resize(Transform):
    """Nearest neighbour; src = dst * src_extent // dst_extent."""

    name = "resize"

    def __init__(self, height: int, width: int):
        self.h = height
        self.w = width

    def output_spec(self, input_spec):
        shape, dtype = _array_spec(input_spec, self.name)
        if len(shape) != 3:
            raise SpecMismatch("resize expects HxWxC input")
        return (self.h, self.w, shape[2]), dtype

    def to_ops(self, input_spec):
        return [_op(L.OP_RESIZE, h=self.h, w=self.w)]


class Opaque(Transform):
    """Arbitrary host callable.  Accepted by the API, rejected by device plans."""

    category = Category.OPAQUE

    def __init__(self, fn, name: str = "opaque", spec_fn=None):
        self._fn = fn
        self.name = name
        self._spec_fn = spec_fn

    def output_spec(self, input_spec):
        if self._spec_fn is not None:
            return self._spec_fn(input_spec)
        return _array_spec(input_spec, self.name)

    def to_ops(self, input_spec):
        raise SpecMismatch(f"opaque transform {self.name!r} cannot run on the device path "
                           "(no CPU fallback); express it with device transforms")


# ---------------------------------------------------------------- extensions

def _pair(size):
    if isinstance(size, int):
        return size, size
    h, w = size
    return int(h), int(w)


class RandomResizedCrop(SourceTransform):
    """Decoder: random scale/aspect window of the real image, bilinear-resized.

    FFCV's RandomResizedCropRGBImageDecoder(output_size, scale, ratio).  The
    window rule is torchvision's get_params with bbox Rng draws; the resample
    is bilinear with half-pixel centres (within +-1 LSB of OpenCV).  Unlike
    RandomCrop it samples inside the image's own (h, w), not the padded canvas.
    """

    name = "random-resized-crop"

    def __init__(self, output_size, scale=(0.08, 1.0), ratio=(3 / 4, 4 / 3)):
        self.h, self.w = _pair(output_size)
        self.scale = (float(scale[0]), float(scale[1]))
        self.ratio = (float(ratio[0]), float(ratio[1]))
        if not (0 < self.scale[0] <= self.scale[1]) or not (0 < self.ratio[0] <= self.ratio[1]):
            raise SpecMismatch("random-resized-crop needs 0 < scale[0] <= scale[1] and 0 < ratio[0] <= ratio[1]")

    def output_spec(self, input_spec):
        if not isinstance(input_spec, ImageSourceSpec):
            raise SpecMismatch(f"{self.name} expects an image field, got {input_spec!r}")
        return (self.h, self.w, input_spec.channels), np.dtype(np.uint8)

    def to_ops(self, input_spec):
        return [_op(L.OP_RRC, h=self.h, w=self.w, scale=self.scale, ratio=self.ratio)]


class CenterCrop(SourceTransform):
    """Decoder: centre square of side int(ratio * min(h, w)), bilinear-resized
    (FFCV CenterCropRGBImageDecoder(output_size, ratio))."""

    name = "center-crop"

    def __init__(self, output_size, ratio: float = 224 / 256):
        self.h, self.w = _pair(output_size)
        self.ratio = float(ratio)
        if not 0 < self.ratio <= 1:
            raise SpecMismatch("center-crop ratio must be in (0, 1]")

    def output_spec(self, input_spec):
        if not isinstance(input_spec, ImageSourceSpec):
            raise SpecMismatch(f"{self.name} expects an image field, got {input_spec!r}")
        return (self.h, self.w, input_spec.channels), np.dtype(np.uint8)

    def to_ops(self, input_spec):
        return [_op(L.OP_CENTERCROP, h=self.h, w=self.w, p=self.ratio)]


_OUT_DT = {np.dtype(np.float32): L.DT_F32, np.dtype(np.float16): L.DT_F16}


def _dtype_code(dtype) -> int:
    import torch

    if dtype in (torch.bfloat16, "bfloat16", "bf16"):
        return L.DT_BF16
    if dtype in (torch.float16, "float16", "f16"):
        return L.DT_F16
    if dtype in (torch.float32, "float32", "f32"):
        return L.DT_F32
    try:
        return _OUT_DT[np.dtype(dtype)]
    except (TypeError, KeyError):
        raise SpecMismatch(f"unsupported output dtype {dtype!r}") from None


class NormalizeImage(Transform):
    """Per-channel (x - mean[c]) / std[c] in f32, stored as float32/float16/bfloat16.

    FFCV's NormalizeImage(mean, std, type).  Half outputs are the RN-even
    rounding of the exact f32 result.
    """

    name = "normalize-image"

    def __init__(self, mean, std, dtype=np.float32):
        self.mean = np.asarray(mean, dtype=np.float32).reshape(-1)
        self.std = np.asarray(std, dtype=np.float32).reshape(-1)
        if self.mean.shape != self.std.shape or not 1 <= len(self.mean) <= 4:
            raise SpecMismatch("normalize-image needs 1..4 matching mean/std values")
        if np.any(self.std == 0):
            raise SpecMismatch("normalize std must be nonzero")
        self.dtype_code = _dtype_code(dtype)

    def output_spec(self, input_spec):
        shape, _ = _array_spec(input_spec, self.name)
        if len(self.mean) not in (1, shape[-1]):
            raise SpecMismatch(f"{len(self.mean)} means for {shape[-1]} channels")
        out = {L.DT_F32: np.dtype(np.float32), L.DT_F16: np.dtype(np.float16), L.DT_BF16: "bfloat16"}
        return shape, out[self.dtype_code]

    def to_ops(self, input_spec):
        shape, _ = _array_spec(input_spec, self.name)
        c = shape[-1]
        m = self.mean if len(self.mean) == c else np.repeat(self.mean, c)
        s = self.std if len(self.std) == c else np.repeat(self.std, c)
        ops = [_op(L.OP_NORMALIZE_PC, mean=[float(x) for x in m], std=[float(x) for x in s])]
        if self.dtype_code != L.DT_F32:
            ops.append(_op(L.OP_CAST, dtype=self.dtype_code))
        return ops


class ToTorchImage(Transform):
    """Batch as (N, C, H, W): channels_last=True is a view over the channels-last
    buffer (no copy); channels_last=False is a contiguous NCHW copy (FFCV's
    ToTorchImage fills a contiguous buffer in that case)."""

    name = "to-torch-image"
    view_only = True

    def __init__(self, channels_last: bool = True):
        self.channels_last = channels_last

    def output_spec(self, input_spec):
        return _array_spec(input_spec, self.name)

    def to_ops(self, input_spec):
        return []


class ToTensor(Transform):
    """No-op: batches are already torch tensors."""

    name = "to-tensor"
    view_only = True

    def output_spec(self, input_spec):
        return _array_spec(input_spec, self.name)

    def to_ops(self, input_spec):
        return []


class ToDevice(ToTensor):
    """No-op: batches are produced in HBM of the loader's device."""

    name = "to-device"

    def __init__(self, device=None, non_blocking: bool = True):
        self.device = device


# FFCV aliases (thin)
SimpleRGBImageDecoder = Decode
RandomResizedCropRGBImageDecoder = RandomResizedCrop
CenterCropRGBImageDecoder = CenterCrop
RandomHorizontalFlip = RandomFlip


# ------------------------------------------------------------- CLI grammar

def _rrc(args):
    h, w = int(args[0]), int(args[1])
    if len(args) >= 6:
        return RandomResizedCrop((h, w), (float(args[2]), float(args[3])), (float(args[4]), float(args[5])))
    return RandomResizedCrop((h, w))


REGISTRY = {
    "decode": lambda a: Decode(),
    "float": lambda a: ToFloat(),
    "normalize": lambda a: Normalize(float(a[0]), float(a[1])),
    "flip": lambda a: RandomFlip(float(a[0]) if a else 0.5),
    "crop": lambda a: RandomCrop(int(a[0]), int(a[1])),
    "resize": lambda a: Resize(int(a[0]), int(a[1])),
    # extensions
    "rrc": _rrc,
    "center": lambda a: CenterCrop((int(a[0]), int(a[1])), float(a[2]) if len(a) > 2 else 224 / 256),
}


def parse_pipeline(spec: str) -> list:
    """``decode|crop:32,32|flip:0.5|normalize:127.5,64`` (+ ``rrc:h,w``, ``center:h,w,r``,
    ``normpc:m0,m1,m2/s0,s1,s2[/f16|bf16]``)."""
    out = []
    for part in spec.split("|"):
        part = part.strip()
        if not part:
            continue
        name, _, argstr = part.partition(":")
        if name == "normpc":
            try:
                fields = argstr.split("/")
                mean = [float(x) for x in fields[0].split(",")]
                std = [float(x) for x in fields[1].split(",")]
                dt = {"f16": np.float16, "bf16": "bfloat16", "f32": np.float32}[fields[2]] if len(fields) > 2 \
                    else np.float32
            except (ValueError, IndexError, KeyError) as e:
                raise SpecMismatch(f"bad arguments for transform {name!r}: {argstr!r}") from e
            out.append(NormalizeImage(mean, std, dt))
            continue
        if name not in REGISTRY:
            raise SpecMismatch(f"unknown transform {name!r}")
        args = [a for a in argstr.split(",") if a] if argstr else []
        try:
            out.append(REGISTRY[name](args))
        except (ValueError, IndexError) as e:
            raise SpecMismatch(f"bad arguments for transform {name!r}: {argstr!r}") from e
    if not out:
        raise SpecMismatch("empty pipeline spec")
    return out


# --------------------------------------------------------------- planning

def input_spec_for_field(f: FieldDescriptor):
    if f.kind == FieldKind.IMAGE:
        return ImageSourceSpec(f.max_height, f.max_width, f.channels)
    if f.kind == FieldKind.FIXED_ARRAY:
        return ArraySourceSpec(tuple(f.array_dims), f.array_dtype)
    raise SpecMismatch(f"field {f.name!r} ({f.kind.name}) cannot feed a transform chain")


def default_chain_for_field(f: FieldDescriptor) -> list:
    return [Decode()] if f.kind == FieldKind.IMAGE else [ArrayRead()]


@dataclass
class CompiledChain:
    ops: list                 # bbx_op records
    specs: list               # per-transform output specs (reference spec propagation)
    nchw_view: bool           # ToTorchImage at the end
    nchw_contiguous: bool = False   # ToTorchImage(channels_last=False): contiguous NCHW copy


def compile_chain(transforms, input_spec) -> CompiledChain:
    """Spec propagation (pipeline.py:312-331 rules and error texts) + lowering."""
    if not transforms:
        raise SpecMismatch("a pipeline needs at least one transform")
    if not isinstance(transforms[0], SourceTransform):
        raise SpecMismatch("the first transform must read from the sample source")
    if any(isinstance(t, SourceTransform) for t in transforms[1:]):
        raise SpecMismatch("source transforms may only appear first")
    specs, ops = [], []
    spec = input_spec
    nchw = contiguous = False
    for t in transforms:
        out = t.output_spec(spec)
        t.prepare(spec, out)
        if t.category == Category.OPAQUE or not hasattr(t, "to_ops"):
            raise SpecMismatch(f"opaque transform {t.name!r} cannot run on the device path "
                               "(no CPU fallback); express it with device transforms")
        if isinstance(t, ToTorchImage):
            nchw = t.channels_last is not None
            contiguous = t.channels_last is False
        elif nchw and not getattr(t, "view_only", False):
            raise SpecMismatch("to-torch-image must be the last transform")
        ops.extend(t.to_ops(spec))
        specs.append(out)
        spec = out
    return CompiledChain(ops, specs, nchw, contiguous)
