"""Image blob codecs: encode side (host, for the writer) and device decode.

Codec ids and payload formats as codecs.py:25-128 of the reference:
RAW = row-major HxWxC bytes; RLE = (u32 count, u8 value) runs; SUBSAMPLE2 =
top-left pixel of every 2x2 block.  Decoding happens on the GPU (K2/K1 in
csrc/kernels.cu); `decode_image` here is the single-blob entry point.

JPEG (codec id 3) is this build's extension (the reference stops at 2,
codecs.py:25-28; its validator rejects codec > 2, format.py:542-543): a
baseline, Huffman-coded, single-scan JFIF file with 1 or 3 components and
sampling factors in {1, 2}, written with restart markers so the device
decoder can give every restart interval its own thread (csrc/jpeg.cu).
Encoding (writer side, offline) goes through Pillow / libjpeg-turbo.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from .errors import DimsExceedMax, SchemaMismatch


class CodecId(enum.IntEnum):
    RAW = 0
    RLE = 1
    SUBSAMPLE2 = 2
    JPEG = 3


@dataclass(frozen=True)
class JpegParams:
    """Writer-side JPEG settings (FFCV's RGBImageField(jpeg_quality=90) analogue)."""
    quality: int = 90
    subsampling: str = "4:2:0"     # "4:4:4" | "4:2:2" | "4:2:0"
    restart_rows: int = 0          # DRI = this many MCU rows (takes precedence when > 0)
    restart_blocks: int = 2        # else DRI = this many MCUs (0 and rows 0: no restart markers)


def encode_jpeg(px: np.ndarray, params: JpegParams | None = None) -> bytes:
    """Baseline JFIF bytes for a u8 (h, w, 1|3) array (Pillow / libjpeg-turbo)."""
    import io

    from PIL import Image

    params = params or JpegParams()
    h, w, c = px.shape
    if c not in (1, 3):
        raise SchemaMismatch(f"jpeg needs 1 or 3 channels, got {c}")
    im = Image.fromarray(px[:, :, 0] if c == 1 else px, "L" if c == 1 else "RGB")
    kw = {"quality": int(params.quality)}
    if c == 3:
        kw["subsampling"] = params.subsampling
    # Restart intervals are the device decoder's unit of parallelism (one
    # thread each); 2 MCUs cost ~1.5% in file size at q90.
    if params.restart_rows:
        kw["restart_marker_rows"] = int(params.restart_rows)
    elif params.restart_blocks:
        kw["restart_marker_blocks"] = int(params.restart_blocks)
    bio = io.BytesIO()
    im.save(bio, "JPEG", **kw)
    return bio.getvalue()


@dataclass(frozen=True)
class ImageBlob:
    height: int
    width: int
    channels: int
    codec: CodecId
    payload: bytes


def subsampled_dims(height: int, width: int) -> tuple[int, int]:
    return (height + 1) // 2, (width + 1) // 2


def decoded_nbytes(blob: ImageBlob) -> int:
    return blob.height * blob.width * blob.channels


def encode_rle(flat: np.ndarray) -> bytes:
    """(count u32 LE, value u8) runs of a flat u8 array."""
    flat = np.ascontiguousarray(flat, dtype=np.uint8).reshape(-1)
    if flat.size == 0:
        return b""
    edges = np.flatnonzero(flat[1:] != flat[:-1]) + 1
    starts = np.r_[0, edges]
    counts = np.diff(np.r_[starts, flat.size]).astype("<u4")
    rec = np.empty(len(starts), dtype=[("n", "<u4"), ("v", "u1")])
    rec["n"] = counts
    rec["v"] = flat[starts]
    return rec.tobytes()


def encode_image(pixels, codec, *, max_height=None, max_width=None, jpeg: JpegParams | None = None) -> ImageBlob:
    px = np.asarray(pixels)
    if px.dtype != np.uint8 or px.ndim != 3:
        raise SchemaMismatch(f"expected a u8 HxWxC array, got {px.dtype} ndim={px.ndim}")
    if 0 in px.shape:
        raise SchemaMismatch("image dims must all be >= 1")
    px = np.ascontiguousarray(px)
    h, w, c = px.shape
    if (max_height is not None and h > max_height) or (max_width is not None and w > max_width):
        raise DimsExceedMax(f"image {h}x{w} exceeds descriptor max {max_height}x{max_width}")
    codec = CodecId(codec)
    if codec == CodecId.RAW:
        payload = px.tobytes()
    elif codec == CodecId.RLE:
        payload = encode_rle(px)
    elif codec == CodecId.JPEG:
        payload = encode_jpeg(px, jpeg)
    else:
        payload = px[::2, ::2].tobytes()
    return ImageBlob(h, w, c, codec, payload)


def decode_image(blob: ImageBlob, out, device: int | None = None) -> None:
    """Decode one blob on the GPU into `out` (codecs.py:91-128 contract).

    `out` is a u8 (h, w, c) buffer: a CUDA torch tensor is written in place on
    its device; a numpy array receives the device result (D2H copy).
    """
    import torch

    from ._lib import check, lib

    h, w, c = blob.height, blob.width, blob.channels
    shape = tuple(out.shape)
    is_torch = isinstance(out, torch.Tensor)
    dt_ok = (out.dtype == torch.uint8) if is_torch else (out.dtype == np.uint8)
    if shape != (h, w, c) or not dt_ok:
        raise SchemaMismatch(f"output buffer must be u8 ({h}, {w}, {c}), got {out.dtype} {shape}")
    payload = bytes(blob.payload)
    buf = ctypes.create_string_buffer(payload, max(len(payload), 1))
    if is_torch:
        if not out.is_cuda or not out.is_contiguous():
            raise SchemaMismatch("decode_image needs a contiguous CUDA tensor or a numpy array")
        dev = out.device.index
        target = out
    else:
        dev = torch.cuda.current_device() if device is None else device
        target = torch.empty((h, w, c), dtype=torch.uint8, device=f"cuda:{dev}")
    check(lib().bbx_decode_image(h, w, c, int(blob.codec), ctypes.addressof(buf), len(payload),
                                 target.data_ptr(), dev))
    if not is_torch:
        out[...] = target.cpu().numpy()
