#pragma once
// image_kernel.cuh — K1 and the helpers shared by every kernel TU.
// sm_100a kernels of the bbox hot path.  See DESIGN.md §4 for the roofline of
// each kernel.  Nothing here is a dense contraction, so no tensor cores: the
// image kernel is an HBM-bound gather/expand.  Every global load is a 16-byte
// vector into shared memory and every store a 16-byte vector of the
// channels-last (NHWC) output.
//
//   K1 image_kernel       Decode (RAW/SUBSAMPLE2/expanded-RLE canvas, zero pad)
//                         + RandomCrop/RandomFlip/Resize remaps + value ops
//                         (ToFloat/Normalize/per-channel/cast), or the bilinear
//                         RandomResizedCrop / CenterCrop decoders.
//                         Reference: pipeline.py:95-231, codecs.py:91-128.
//   K2 rle_expand_kernel  codecs.py:101-114 (RLE runs -> dense canvas), with
//                         the reference's error semantics as a status word.
//   K3 scalar_gather      loader.py:333-335 (label[b] = column[idx[b]]).
//   K3' array_kernel      ArrayRead (pipeline.py:128-129) + chain.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <algorithm>
#include <map>
#include <type_traits>
#include <mutex>

#include "bbx_internal.h"

namespace bbx {

constexpr int VAL_GENERIC = 100;   // template tag: runtime choice between VAL_FMA and VAL_DIRECT

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Output-to-input coordinate through the remaps, applied last-to-first.
// Every remap is monotone per axis (crop: shift, flip: reversal, nearest
// resize: floor scaling), so the composition is monotone too.
__device__ __forceinline__ int back_y(const PlanDev& P, const int32_t* prm, int y) {
  for (int i = P.n_remaps - 1; i >= 0; --i) {
    const Remap& m = P.remaps[i];
    if (m.kind == BBX_OP_CROP) y += prm[m.prm];
    else if (m.kind == BBX_OP_RESIZE) y = (int)(((int64_t)y * m.in_h) / m.out_h);
  }
  return y;
}
__device__ __forceinline__ int back_x(const PlanDev& P, const int32_t* prm, int x) {
  for (int i = P.n_remaps - 1; i >= 0; --i) {
    const Remap& m = P.remaps[i];
    if (m.kind == BBX_OP_CROP) x += prm[m.prm + 1];
    else if (m.kind == BBX_OP_FLIP) { if (prm[m.prm]) x = m.in_w - 1 - x; }
    else if (m.kind == BBX_OP_RESIZE) x = (int)(((int64_t)x * m.in_w) / m.out_w);
  }
  return x;
}

// Bilinear axis (extension; identical integer rule in oracle/bbx_oracle.c
// lin_axis): half-pixel centres, replicated border, 11-bit weight of i1.
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t magic) { return __umulhi(n, magic); }

__device__ __forceinline__ void lin_axis(int o, int out_n, int in_n, bool fits32, uint32_t magic, int& i0, int& i1,
                                         int& w1) {
  int64_t num = (int64_t)(2 * o + 1) * in_n - out_n, den = 2 * (int64_t)out_n;
  if (num <= 0) { i0 = 0; i1 = 0; w1 = 0; return; }
  int64_t q, r;
  if (magic) {   // den is the plan's 2*canvas extent: exact reciprocal multiply
    uint32_t q32 = fast_div((uint32_t)num, magic);
    uint32_t r32 = (uint32_t)num - q32 * (uint32_t)den;
    if (q32 >= (uint32_t)(in_n - 1)) { i0 = in_n - 1; i1 = in_n - 1; w1 = 0; return; }
    i0 = (int)q32; i1 = (int)q32 + 1;
    w1 = (int)fast_div(r32 * 2048u + (uint32_t)(den >> 1), magic);
    return;
  }
  if (fits32) {
    uint32_t n32 = (uint32_t)num, d32 = (uint32_t)den;
    uint32_t q32 = n32 / d32;
    q = q32; r = n32 - q32 * d32;
  } else {
    q = num / den; r = num - q * den;
  }
  if (q >= in_n - 1) { i0 = in_n - 1; i1 = in_n - 1; w1 = 0; return; }
  i0 = (int)q; i1 = (int)q + 1;
  w1 = fits32 ? (int)(((uint32_t)r * 2048u + (uint32_t)(den >> 1)) / (uint32_t)den)
              : (int)((r * 2048 + den / 2) / den);
}

__device__ __forceinline__ float to_f32(const uint8_t* p, int dt) {
  switch (dt) {
    case BBX_U8: return (float)*p;
    case BBX_I64: { long long v; memcpy(&v, p, 8); return __ll2float_rn(v); }
    case BBX_F32: { float v; memcpy(&v, p, 4); return v; }
    case BBX_F64: { double v; memcpy(&v, p, 8); return __double2float_rn(v); }
  }
  return 0.f;
}

// Value ops in strict IEEE f32 (pipeline.py:158-160: one subtract, one divide).
__device__ __forceinline__ float apply_vops(const PlanDev& P, float v, int k) {
  for (int i = 0; i < P.n_vops; ++i) v = __fdiv_rn(__fsub_rn(v, P.vop_mean[i][k & 3]), P.vop_std[i][k & 3]);
  return v;
}
// Same results, without the divide: q0 = d * RN(1/s), one exact-residual
// correction.  Used only when the host proved it equal to the IEEE quotient
// for every reachable input of the plan (engine.cpp: verify_fma_normalize).
__device__ __forceinline__ float apply_vops_fma(const PlanDev& P, float v, int k) {
  for (int i = 0; i < P.n_vops; ++i) {
    float d = __fsub_rn(v, P.vop_mean[i][k & 3]);
    float inv = P.vop_inv[i][k & 3];
    float q0 = __fmul_rn(d, inv);
    float r = __fmaf_rn(-q0, P.vop_std[i][k & 3], d);
    v = __fmaf_rn(r, inv, q0);
  }
  return v;
}

template <typename T> __device__ __forceinline__ T cvt_out(float v);
template <> __device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <> __device__ __forceinline__ __half cvt_out<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ uint8_t cvt_out<uint8_t>(float v) { return (uint8_t)v; }

template <typename OutT, int kVal>
__device__ __forceinline__ OutT value_generic(const PlanDev& P, uint32_t b, int k) {
  if constexpr (kVal == VAL_COPY) return (OutT)b;
  else return cvt_out<OutT>(P.value_mode == VAL_DIRECT ? apply_vops(P, (float)b, k) : apply_vops_fma(P, (float)b, k));
}

// Shared-memory layout of the image kernel (host + device).
__host__ __device__ inline int align_up(int v, int a) { return (v + a - 1) / a * a; }

__host__ __device__ inline int out_size(const PlanDev& P) {
  return P.out_dtype == BBX_U8 ? 1 : (P.out_dtype == BBX_F32 ? 4 : 2);
}

__host__ __device__ inline SmemLayout img_layout(const PlanDev& P) {
  SmemLayout L;
  const bool res = P.src_kind == SRC_RESAMPLE;
  const int R = P.rows_per_tile;
  L.nslot = res ? 2 * R : R;
  L.span_pad = align_up(P.src_row_w * P.channels, 16) + 32;
  L.hrow_pad = align_up(P.out_w * P.channels * (res ? 4 : 1), 16) + 16;
  L.xt_off = 0;
  L.meta_off = align_up(P.out_w * 4, 16);
  // meta: slot_row[nslot], shift[nslot], row_a[R], row_b[R], row_wy[R] (int32)
  const int lut = P.value_mode == VAL_LUT ? align_up(P.channels * 256 * out_size(P), 16) : 0;
  L.src_off = L.meta_off + align_up((2 * L.nslot + 3 * R) * 4, 16) + lut;
  L.h_off = L.src_off + L.nslot * L.span_pad;
  L.total = L.h_off + L.nslot * L.hrow_pad;
  return L;
}
__host__ __device__ inline int lut_off(const PlanDev& P) {
  return P.lay.meta_off + align_up((2 * P.lay.nslot + 3 * P.rows_per_tile) * 4, 16);
}

// Per-sample tables written by the prologue (u32 words, tab_stride per sample):
//   [0] col_lo  [1] col_hi  [2..3] pad
//   [4 .. 4+OWp)          column table xt (encoded, see below)
//   per tile t (TM words): nvalid, slot_row[nslot], row_a[R], row_b[R], row_wy[R]
__host__ __device__ inline int tab_owp(const PlanDev& P) { return align_up(P.out_w, 4); }
__host__ __device__ inline int tab_tm(const PlanDev& P) {
  const int nslot = P.rows_per_tile * (P.src_kind == SRC_RESAMPLE ? 2 : 1);
  return align_up(1 + nslot + 3 * P.rows_per_tile, 4);
}
__host__ __device__ inline int tab_stride(const PlanDev& P) { return 4 + tab_owp(P) + P.tiles_per_sample * tab_tm(P); }

// Source-row addressing of one sample (codec / staging dependent).
struct SrcRows {
  const uint8_t* base;
  int64_t rstride;
  int sh, rows;
};
__device__ __forceinline__ SrcRows src_rows_of(const PlanDev& P, const LaunchArgs& A, const SampleDesc* d, int s) {
  SrcRows S;
  const int C = P.channels, w = d->w, h = d->h;
  if (d->codec == CODEC_RLE || d->codec == CODEC_JPEG) {   // decoded into scratch by K2 / J1-J4
    S.base = A.scratch + (size_t)s * P.scratch_bytes; S.sh = 0;
    S.rstride = d->codec == CODEC_JPEG ? jpeg_scratch_pitch(w, C) : (int64_t)w * C;
  } else if (d->flags & kDescWindowed) {
    // only the rows/columns the chain reads were staged: a virtual origin makes
    // every in-window image coordinate address its staged byte
    S.rstride = d->wstride; S.sh = 0;
    S.base = A.payload + d->src - (int64_t)d->wy0 * S.rstride - (int64_t)d->wx0 * C;
  } else {
    S.base = A.payload + d->src; S.sh = d->codec == CODEC_SUB2 ? 1 : 0;
    S.rstride = (int64_t)(S.sh ? (w + 1) >> 1 : w) * C;
  }
  S.rows = S.sh ? (h + 1) >> 1 : h;
  return S;
}

// --------------------------------------------------------------- K1 prologue
// One CTA per sample: the remap/resample geometry that every tile of the
// sample shares -- the encoded column table and, per tile, the source-row
// slots -- computed once instead of once per tile.
//   xt (bilinear): byte offset of tap 0 (16 b) | 11-bit weight of tap 1 << 16 | same-column bit << 28
//   xt (nearest):  byte offset, or 0xFFFFFFFF for a zero-padding column
template <bool kRes>
__global__ void __launch_bounds__(kThreads) sample_tables_kernel(const PlanDev P, const LaunchArgs A) {
  const int s = blockIdx.x;
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  if (d->skip) return;
  const int32_t* prm = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(d) + kDescHeader);
  const int OW = P.out_w, OH = P.out_h, C = P.channels, h = d->h, w = d->w, tid = threadIdx.x;
  const SrcRows S = src_rows_of(P, A, d, s);
  const int sh = S.sh;
  extern __shared__ __align__(16) int tsm[];
  int* xraw = tsm;                      // OW
  int* ya = xraw + OW;                  // OH each
  int* yb = ya + OH;
  int* wyv = yb + OH;
  __shared__ int s_clo, s_chi;
  uint32_t* T = A.tables + (size_t)s * P.tab_stride;
  const int top = kRes ? prm[0] : 0, left = kRes ? prm[1] : 0, ch = kRes ? prm[2] : 0, cw = kRes ? prm[3] : 0;
  for (int ox = tid; ox < OW; ox += kThreads) xraw[ox] = back_x(P, prm, ox);
  for (int r = tid; r < OH; r += kThreads) {
    if constexpr (kRes) {
      int cy = back_y(P, prm, r), y0, y1, wy;
      lin_axis(cy, P.canvas_h, ch, P.lin32, P.liny_magic, y0, y1, wy);
      ya[r] = (top + y0) >> sh; yb[r] = (top + y1) >> sh; wyv[r] = wy;
    } else {
      int cy = back_y(P, prm, r);
      ya[r] = cy < h ? (cy >> sh) : -1;
    }
  }
  __syncthreads();
  if (tid == 0) {   // the composed maps are monotone: the end columns span the range
    int xa = xraw[0], xb = xraw[OW - 1], clo, chi;
    if constexpr (kRes) {
      int a0, a1, aw, b0, b1, bw;
      lin_axis(min(xa, xb), P.canvas_w, cw, P.lin32, P.linx_magic, a0, a1, aw);
      lin_axis(max(xa, xb), P.canvas_w, cw, P.lin32, P.linx_magic, b0, b1, bw);
      clo = (left + a0) >> sh; chi = (left + b1) >> sh;
    } else {
      clo = min(xa, xb) >> sh; chi = min(max(xa, xb), w - 1) >> sh;   // clo > chi: all padding
    }
    s_clo = clo; s_chi = chi;
    T[0] = (uint32_t)clo; T[1] = (uint32_t)chi;
  }
  __syncthreads();
  const int col_lo = s_clo;
  uint32_t* xt = T + 4;
  for (int ox = tid; ox < OW; ox += kThreads) {
    const int cx = xraw[ox];
    if constexpr (kRes) {
      int x0, x1, wx;
      lin_axis(cx, P.canvas_w, cw, P.lin32, P.linx_magic, x0, x1, wx);
      int c0 = (left + x0) >> sh, c1 = (left + x1) >> sh;
      xt[ox] = (uint32_t)((c0 - col_lo) * C) | ((uint32_t)wx << 16) | (c1 == c0 ? (1u << 28) : 0u);
    } else {
      xt[ox] = cx < w ? (uint32_t)(((cx >> sh) - col_lo) * C) : 0xFFFFFFFFu;
    }
  }
  // per tile: contiguous source-row range -> slots when it fits, else one
  // slot per (output row, tap)
  const int Rt = P.rows_per_tile, nslot = kRes ? 2 * Rt : Rt, TM = tab_tm(P);
  for (int t = tid; t < P.tiles_per_sample; t += kThreads) {
    uint32_t* M = T + 4 + tab_owp(P) + (size_t)t * TM;
    int* slot = reinterpret_cast<int*>(M + 1);
    int* ra = slot + nslot;
    int* rb = ra + Rt;
    int* rw = rb + Rt;
    const int r0 = t * Rt, R = min(Rt, OH - r0);
    int lo = ya[r0], hi = kRes ? yb[r0 + R - 1] : ya[r0 + R - 1];
    if (!kRes && lo < 0) { lo = hi = -1; }
    if (!kRes && hi < 0) {
      hi = -1;
      for (int r = R - 1; r >= 0; --r) if (ya[r0 + r] >= 0) { hi = ya[r0 + r]; break; }
    }
    const bool contiguous = lo >= 0 && hi >= lo && hi - lo + 1 <= nslot;
    if (contiguous) {
      M[0] = (uint32_t)(hi - lo + 1);
      for (int j = 0; j < nslot; ++j) slot[j] = (lo + j <= hi && lo + j < S.rows) ? lo + j : -1;
      for (int r = 0; r < R; ++r) {
        ra[r] = ya[r0 + r] >= 0 ? ya[r0 + r] - lo : -1;
        if constexpr (kRes) { rb[r] = yb[r0 + r] - lo; rw[r] = wyv[r0 + r]; }
      }
    } else {
      M[0] = (uint32_t)nslot;
      for (int j = 0; j < nslot; ++j) slot[j] = -1;
      for (int r = 0; r < R; ++r) {
        if constexpr (kRes) {
          slot[2 * r] = ya[r0 + r]; slot[2 * r + 1] = yb[r0 + r];
          ra[r] = 2 * r; rb[r] = 2 * r + 1; rw[r] = wyv[r0 + r];
        } else {
          slot[r] = ya[r0 + r];
          ra[r] = ya[r0 + r] >= 0 ? r : -1;
        }
      }
    }
  }
}

// V: vertical pass + value ops + 16-byte stores for R output rows whose
// horizontally resampled source rows sit in hbuf (row_a / row_b = hbuf rows,
// -1 = zero row).  Each thread owns one group of kC x 16 B of output (V
// pixels), so the channel of every element is a compile-time constant.
template <typename OutT, bool kRes, int kVal, int kC, bool kVec>
__device__ __forceinline__ void vpass(const PlanDev& P, const uint8_t* hbuf, int hrow_pad, const int* row_a,
                                      const int* row_b, const int* row_wy, int R, OutT* out, const OutT* lut,
                                      int tid) {
  constexpr int V = kVec ? (16 / (int)sizeof(OutT)) : 1;
  const int C = kC > 0 ? kC : P.channels;
  const int OW = P.out_w;
  const int rowlen = OW * C;
  auto val = [&](uint32_t b, int k) -> OutT {
    if constexpr (kVal == VAL_LUT) return lut[k * 256 + b];
    else return value_generic<OutT, kVal>(P, b, k);
  };
  if constexpr (kC > 0) {
    // group = V pixels = kC vectors of V elements; element i of vector j has channel (j*V+i) % kC
    const int gpr = OW / V;                     // full groups per row
    const int ngroups = R * gpr;
    for (int idx = tid; idx < ngroups; idx += kThreads) {
      int r = (kVec && P.gpr_magic) ? (int)fast_div((uint32_t)idx, P.gpr_magic) : idx / gpr;
      int g = idx - r * gpr;
      int e0 = g * V * kC;
      int a = row_a[r];
      OutT* orow = out + (size_t)r * rowlen + e0;
#pragma unroll
      for (int j = 0; j < kC; ++j) {
        union { OutT v[V]; uint4 u; } pk;
        if constexpr (kRes) {
          const uint32_t* h0 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)a * hrow_pad) + e0 + j * V;
          const uint32_t* h1 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)row_b[r] * hrow_pad) + e0 + j * V;
          const uint32_t wy1 = (uint32_t)row_wy[r], wy0 = 2048u - wy1;
          uint32_t t0[V], t1[V];
          if constexpr (V % 4 == 0) {
#pragma unroll
            for (int i = 0; i < V; i += 4) {
              uint4 x = *reinterpret_cast<const uint4*>(h0 + i), y = *reinterpret_cast<const uint4*>(h1 + i);
              t0[i] = x.x; t0[i + 1] = x.y; t0[i + 2] = x.z; t0[i + 3] = x.w;
              t1[i] = y.x; t1[i + 1] = y.y; t1[i + 2] = y.z; t1[i + 3] = y.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i) { t0[i] = h0[i]; t1[i] = h1[i]; }
          }
#pragma unroll
          for (int i = 0; i < V; ++i) pk.v[i] = val((wy0 * t0[i] + wy1 * t1[i] + (1u << 21)) >> 22, (j * V + i) % kC);
        } else {
          uint8_t bytes[V];
          if (a < 0) {
#pragma unroll
            for (int i = 0; i < V; ++i) bytes[i] = 0;
          } else {
            const uint8_t* h0 = hbuf + (size_t)a * hrow_pad + e0 + j * V;
            if constexpr (V == 16) *reinterpret_cast<uint4*>(bytes) = *reinterpret_cast<const uint4*>(h0);
            else if constexpr (V == 8) *reinterpret_cast<uint2*>(bytes) = *reinterpret_cast<const uint2*>(h0);
            else if constexpr (V == 4) *reinterpret_cast<uint32_t*>(bytes) = *reinterpret_cast<const uint32_t*>(h0);
            else {
#pragma unroll
              for (int i = 0; i < V; ++i) bytes[i] = h0[i];
            }
          }
#pragma unroll
          for (int i = 0; i < V; ++i) pk.v[i] = val(bytes[i], (j * V + i) % kC);
        }
        if constexpr (kVec) *reinterpret_cast<uint4*>(orow + j * V) = pk.u;
        else orow[j * V] = pk.v[0];
      }
    }
    // tail columns (OW % V) element-wise
    const int tail0 = gpr * V;
    if (tail0 < OW) {
      const int tl = (OW - tail0) * C;
      for (int idx = tid; idx < R * tl; idx += kThreads) {
        int r = idx / tl, q = tail0 * C + (idx - r * tl);
        int k = q % C, a = row_a[r];
        uint32_t b;
        if constexpr (kRes) {
          const uint32_t* h0 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)a * hrow_pad);
          const uint32_t* h1 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)row_b[r] * hrow_pad);
          b = ((2048u - (uint32_t)row_wy[r]) * h0[q] + (uint32_t)row_wy[r] * h1[q] + (1u << 21)) >> 22;
        } else {
          b = hbuf[(size_t)max(a, 0) * hrow_pad + q];
          if (a < 0) b = 0u;
        }
        out[(size_t)r * rowlen + q] = val(b, k);
      }
    }
  } else {
    // dynamic channel count: element-wise
    for (int idx = tid; idx < R * rowlen; idx += kThreads) {
      int r = idx / rowlen, q = idx - r * rowlen;
      int k = q % C, a = row_a[r];
      uint32_t b;
      if constexpr (kRes) {
        const uint32_t* h0 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)a * hrow_pad);
        const uint32_t* h1 = reinterpret_cast<const uint32_t*>(hbuf + (size_t)row_b[r] * hrow_pad);
        b = ((2048u - (uint32_t)row_wy[r]) * h0[q] + (uint32_t)row_wy[r] * h1[q] + (1u << 21)) >> 22;
      } else {
        b = hbuf[(size_t)max(a, 0) * hrow_pad + q];
        if (a < 0) b = 0u;
      }
      out[(size_t)r * rowlen + q] = val(b, k);
    }
  }
}

// --------------------------------------------------------------------- K1
// grid = (tiles_per_sample, count); CTA = 256 threads; a tile = R output rows.
//
//  A. the tile's slice of the prologue tables -> smem (column table, row
//     slots) and, for normalize chains, the exact u8 -> output LUT.
//  B. every needed source row segment -> smem, 16-byte vector loads.
//  H. horizontal pass, once per staged row: u8 (nearest) or the 2-tap
//     fixed-point sum (bilinear, u32) for every output column and channel.
//  V. vertical pass + value LUT + store: each thread owns one group of
//     kC x 16 B of output (V pixels), so the channel of every element is a
//     compile-time constant; 16-byte coalesced NHWC stores.
template <typename OutT, bool kRes, int kVal, int kC, bool kVec>
__global__ void __launch_bounds__(kThreads, 4) image_kernel(const PlanDev P, const LaunchArgs A) {
  constexpr int V = kVec ? (16 / (int)sizeof(OutT)) : 1;
  const int s = blockIdx.y;
  if (blockIdx.x == 0 && (int)threadIdx.x < A.sc.n_fields)   // the batch's scalar fields, once per sample
    A.sc.outs[threadIdx.x][s] = A.sc.cols[threadIdx.x][A.sc.idx[s]];
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  if (d->skip) return;
  const int C = kC > 0 ? kC : P.channels;
  const int tile = blockIdx.x;
  const int r0 = tile * P.rows_per_tile;
  const int R = min(P.rows_per_tile, P.out_h - r0);
  if (R <= 0) return;
  const int OW = P.out_w;
  const int rowlen = OW * C;
  const int tid = threadIdx.x;
  const SrcRows S = src_rows_of(P, A, d, s);

  extern __shared__ __align__(16) uint8_t smem[];
  const SmemLayout& L = P.lay;
  uint32_t* xt = reinterpret_cast<uint32_t*>(smem + L.xt_off);
  int* slot_row = reinterpret_cast<int*>(smem + L.meta_off);   // source row of slot j, -1 = none
  int* s_shift = slot_row + L.nslot;                            // 16-byte misalignment of slot j
  int* row_a = s_shift + L.nslot;                               // per output row: slot (-1: zero row)
  int* row_b = row_a + P.rows_per_tile;                         // bilinear second slot
  int* row_wy = row_b + P.rows_per_tile;
  OutT* lut = reinterpret_cast<OutT*>(smem + lut_off(P));
  uint8_t* srcbuf = smem + L.src_off;
  uint8_t* hbuf = smem + L.h_off;

  // ---- A: tables
  const uint32_t* T = A.tables + (size_t)s * P.tab_stride;
  const int col_lo = (int)T[0], col_hi = (int)T[1];
  const int span_bytes = col_hi >= col_lo ? (col_hi - col_lo + 1) * C : 0;
  for (int i = tid; i < OW; i += kThreads) xt[i] = T[4 + i];
  const uint32_t* M = T + 4 + tab_owp(P) + (size_t)tile * tab_tm(P);
  const int nvalid = (int)M[0];
  if (tid < L.nslot) { slot_row[tid] = (int)M[1 + tid]; s_shift[tid] = 0; }
  if (tid < 3 * P.rows_per_tile) row_a[tid] = (int)M[1 + L.nslot + tid];   // row_a, row_b, row_wy
  if constexpr (kVal == VAL_LUT) {
    const uint4* g = reinterpret_cast<const uint4*>(A.lut);
    uint4* l4 = reinterpret_cast<uint4*>(lut);
    const int n16 = C * 256 * (int)sizeof(OutT) / 16;
    for (int i = tid; i < n16; i += kThreads) l4[i] = g[i];
  }
  __syncthreads();

  // ---- B: stage source row segments (warp per slot, 16 B vectors)
  const int lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < nvalid; j += kThreads / 32) {
    int srow = slot_row[j];
    if (srow < 0 || span_bytes == 0) continue;
    const uint8_t* src = S.base + (int64_t)srow * S.rstride + (int64_t)col_lo * C;
    uintptr_t a = reinterpret_cast<uintptr_t>(src);
    uintptr_t a0 = a & ~(uintptr_t)15;
    int shift = (int)(a - a0);
    int n16 = (shift + span_bytes + 15) >> 4;
    uint8_t* dst = srcbuf + (size_t)j * L.span_pad;
    const uint8_t* s0 = reinterpret_cast<const uint8_t*>(a0);
    for (int c = lane; c < n16; c += 32) *reinterpret_cast<uint4*>(dst + 16 * c) = ld_nc_v4(s0 + 16 * c);
    if (lane == 0) s_shift[j] = shift;
  }
  __syncthreads();

  // ---- H: horizontal pass; a thread owns one output column (its table entry
  // decoded once) and walks the slots; short rows put several threads per column
  {
    const int ncg = P.h_tpc;                        // threads per column
    for (int c0 = tid; c0 < OW * ncg; c0 += kThreads) {
      const int j0 = P.ow_magic ? (int)fast_div((uint32_t)c0, P.ow_magic) : c0 / OW;
      const int ox = c0 - j0 * OW;
      const uint32_t e = xt[ox];
      if constexpr (kRes) {
        const int off0 = (int)(e & 0xFFFFu), wx = (int)((e >> 16) & 0xFFFu);
        const int off1 = (e >> 28) ? off0 : off0 + C;
        const uint32_t w0 = 2048u - (uint32_t)wx, w1 = (uint32_t)wx;
        for (int j = j0; j < nvalid; j += ncg) {
          if (slot_row[j] < 0) continue;
          const uint8_t* row = srcbuf + j * L.span_pad + s_shift[j];
          uint32_t* hr = reinterpret_cast<uint32_t*>(hbuf + j * L.hrow_pad) + ox * C;
#pragma unroll
          for (int k = 0; k < (kC > 0 ? kC : 1); ++k) hr[k] = w0 * row[off0 + k] + w1 * row[off1 + k];
          if constexpr (kC == 0)
            for (int k = 1; k < C; ++k) hr[k] = w0 * row[off0 + k] + w1 * row[off1 + k];
        }
      } else {
        const bool pad = e == 0xFFFFFFFFu;
        const uint32_t eo = pad ? 0u : e;    // never form an out-of-window smem address
        for (int j = j0; j < nvalid; j += ncg) {
          if (slot_row[j] < 0) continue;
          const uint8_t* row = srcbuf + j * L.span_pad + s_shift[j];
          uint8_t* hr = hbuf + j * L.hrow_pad + ox * C;
#pragma unroll
          for (int k = 0; k < (kC > 0 ? kC : 1); ++k) { uint8_t v = row[eo + k]; hr[k] = pad ? 0 : v; }
          if constexpr (kC == 0)
            for (int k = 1; k < C; ++k) { uint8_t v = row[eo + k]; hr[k] = pad ? 0 : v; }
        }
      }
    }
  }
  __syncthreads();

  vpass<OutT, kRes, kVal, kC, kVec>(P, hbuf, L.hrow_pad, row_a, row_b, row_wy, R,
        reinterpret_cast<OutT*>(A.out) + ((size_t)s * P.out_h + r0) * rowlen, lut, tid);
}

// ------------------------------------------------------- K1 (column walker)
// Bilinear decoders (RandomResizedCrop / CenterCrop), 3 channels.
//
// Persistent CTAs (SMs x resident CTAs) walk the batch's tiles (tile =
// rows_per_tile output rows of one sample), taking runs of cw_run consecutive
// tiles from a global ticket counter (the launch's last fetch re-zeroes it), so
// SMs that drew cheap samples take more.  A CTA is one copy warp plus
// ceil(OW / 64) compute warps; compute thread x owns output columns 2x, 2x + 1 of
// EVERY tile the CTA takes, so its per-column state survives from tile to tile of
// a sample.
//
// Copy warp: takes the tickets (the next run's is fetched while the current run is
// handed out); per tile, once the compute warps have released the stage ("empty"
// mbarrier), it moves the tile's source rows into it with cp.async.bulk (TMA 1-D,
// completion counted in bytes on the stage's "full" mbarrier: one copy per row when
// whole-row copies would move >= 25 % more than the window, else one copy for the
// row range), and while they are in flight writes the tile's geometry into a ring
// entry: on a sample's first tile its column parameters (the compute threads derive
// their own two columns' taps from them), per output row the smem offsets of its
// even and odd source rows, the odd weight and the new-row flags; the arrive on
// "full" comes after.  It also gathers the batch's scalar fields with tile 0 of each
// sample.
//
// Compute: the 2-tap horizontal sums of a source row are formed when the row
// first appears for its parity (even / odd absolute row: the two taps of an
// output row are always one of each), with byte-pair dot products (dp2a) on
// funnel-shifted words, and kept in registers (h_even, h_odd per value).  The
// copy warp mirrors which rows the compute warps hold and flags, per output row,
// the parities whose row is new, so the compute loop does no tag bookkeeping.
// The vertical blend is two integer multiply-adds per value,
//     s = 4 w_even h_even + 4 w_odd h_odd + 2^23 = 4 (w_even h_even + w_odd h_odd + 2^21),  u = s >> 24,
// the same integer the tile kernel / oracle form ((w0 h0 + w1 h1 + 2^21) >> 22,
// bit for bit).  When a sample's row stride is a multiple of 4 every staged row
// has the same byte phase mod 4, so the column offsets carry it and a tap's
// bytes are three aligned shared loads at row + column offset.  u -> output:
// f16 / bf16 through a per-channel f32 affine map fma(u, A, B) that the host
// proved equal to the exact value table for all 256 inputs (packed f32x2 math,
// no shared-memory table), else the table; packed 32-bit stores.
enum CwMode : int { CW_COPY = 0, CW_LUT = 1, CW_AFFINE = 2 };
constexpr int kK1Unroll = 2;                // row loop unroll (A/B: 1 / 2 / 4 -> 45.3 / 44.9 / 45.1 us under ncu)
// one bulk copy per source row when whole-row copies would move >= 25 % more bytes than
// the window, else one copy of the whole row range (A/B: thresholds 5/4, 6/4, 8/4 take
// the same time; 5/4 keeps the DRAM read side at 1.18x the window vs 1.32x at 8/4)
constexpr int kCwPerRowNum = 5, kCwPerRowDen = 4;
constexpr uint32_t kCwFake = 0xFFFEu;       // a parity with weight 0 in this output row (never a real row: heights < 0xFFFE)
constexpr uint32_t kCwNone = 0xFFFFFFFFu;   // no source row held (start of a sample)

__host__ __device__ inline int cw_span_pad(const PlanDev& P) { return align_up(P.src_row_w * P.channels, 16) + 32; }
__host__ __device__ inline int cw_lut_bytes(const PlanDev& P) {
  return (P.value_mode == VAL_LUT && !P.cw_affine) ? align_up(P.channels * 256 * out_size(P), 16) : 0;
}
__host__ __device__ inline int cw_bar_off(const PlanDev& P) { return cw_lut_bytes(P); }
__host__ __device__ inline int cw_stage_off(const PlanDev& P) { return cw_bar_off(P) + 16 * kCwStages; }
// ring entry (stages + 1 of them): header (16 B: first row, sample, live, new-sample) | the sample's column parameters (32 B) |
// per output row uint4 {even row's stage offset, odd row's stage offset, tag_even | tag_odd << 16, 4 * w_odd}
__host__ __device__ inline int cw_tap_off(const PlanDev&) { return 48; }
__host__ __device__ inline int cw_stage_meta(const PlanDev& P) { return cw_tap_off(P) + 16 * P.rows_per_tile; }
__host__ __device__ inline int cw_src_stage(const PlanDev& P) { return P.cw_slots * cw_span_pad(P); }
__host__ __device__ inline int cw_smem_bytes(const PlanDev& P) {
  return cw_stage_off(P) + (kCwStages + 1) * cw_stage_meta(P) + kCwStages * cw_src_stage(P);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* m, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W%=;\n}" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint4 lds_v4(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(tx) : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned ends, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
// c + a.lo16 * b.byte0 + a.hi16 * b.byte1 (signed 16-bit weights, unsigned bytes); _hi: bytes 2, 3
__device__ __forceinline__ int dp2a_lo(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp2a.hi.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
// (x - y) and fma(x, a, b) on f32 pairs, one instruction each (FADD2 / FFMA2; .rn: never contracted)
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long x, unsigned long long y) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  return d;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long x, unsigned long long a,
                                                     unsigned long long b) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(a), "l"(b));
  return d;
}
// bits of the float 2^23 + (s >> 24): one IMAD.HI on the FMA pipe
__device__ __forceinline__ uint32_t u8_magic(uint32_t s) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, 256, 0x4B000000;" : "=r"(d) : "r"(s));
  return d;
}
template <typename OutT> __device__ __forceinline__ uint32_t cvt_pack2(unsigned long long y);
template <> __device__ __forceinline__ uint32_t cvt_pack2<__half>(unsigned long long y) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "r"((uint32_t)(y >> 32)), "r"((uint32_t)y));
  return d;
}
template <> __device__ __forceinline__ uint32_t cvt_pack2<__nv_bfloat16>(unsigned long long y) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "r"((uint32_t)(y >> 32)), "r"((uint32_t)y));
  return d;
}

template <typename OutT, int kMode>
__global__ void __launch_bounds__(9 * 32, 2) image_cw_kernel(const PlanDev P, const LaunchArgs A) {
  constexpr int C = 3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncw = P.cw_warps;                          // compute warps 0..ncw-1; warp ncw issues the copies
  const int OW = P.out_w, tps = P.tiles_per_sample, Rt = P.rows_per_tile;
  const int nslot = P.cw_slots, meta = cw_stage_meta(P), sbytes = cw_src_stage(P), span_pad = cw_span_pad(P);
  const int tap_off = cw_tap_off(P);
  // tickets: the first `nrun` hand out runs of cw_run consecutive tiles (sample-major
  // order), the last ~2 x grid tiles go out one by one (a short tail; half tiles were
  // measured slower, 43 -> 50 us: each half re-sums its first rows and the column
  // table; handing out the tallest crop windows first made no difference); a CTA's
  // first ticket is its block index, the rest come from a global counter
  const int total = A.count * tps, G = gridDim.x;
  const int run = P.cw_run, tail = min(total, 2 * G), nrun = (total - tail) / run, head = nrun * run;
  const int ntickets = nrun + (total - head);
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NS = kCwStages, NR = kCwStages + 1;   // source stages; geometry ring entries
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + cw_bar_off(P));   // full[NS], empty[NS]
  uint64_t* empty = full + NS;
  uint8_t* metas = smem + cw_stage_off(P);              // geometry ring: tile k uses entry k % NR
  const uint32_t stage0 = (uint32_t)(cw_stage_off(P) + NR * meta);   // source rows: tile k uses stage k % NS
  uint8_t* stages = smem + stage0;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], ncw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();                                   // barriers initialised

  if (warp == ncw) {
    // ---- copy warp: tile k's geometry -> ring entry k % NR (free: iteration
    // k - 1 waited for tile k - 1 - NS), then, once the compute warps have
    // released tile k - NS's stage, its source rows -> stage k % NS (nslot <= 32)
    int k = 0, m = 0, b = 0, ph = 0;                   // ph: parity of stage b's use count
    int left = 0, s = 0, tile = 0, t_id = 0;           // the run being handed out: tiles left, next tile
    int cur_s = -1, col_lo = 0, span_bytes = 0;        // the sample whose column table was last written
    bool aligned = false;                              // its rows share one byte phase mod 4
    int bx0 = 0, bxs = 1, by0 = 0;                     // its x / y maps when they are affine (no Resize)
    uint32_t held_e = kCwNone, held_o = kCwNone;       // mirror: the source rows whose sums the compute warps hold
    int loaded_s = -1, top = 0, ch = 0;                // the sample whose descriptor fields are cached below
    bool s_skip = true;
    SrcRows S{};
    bool affine = true;                                // crops / flips only: back_x, back_y are +-1 slopes
    for (int i = 0; i < P.n_remaps; ++i) affine = affine && P.remaps[i].kind != BBX_OP_RESIZE;
    // the next run's ticket is fetched while the current run is handed out
    unsigned long long next_u = blockIdx.x;
    for (;; ++k, m = m == NR - 1 ? 0 : m + 1) {
      if (k > 0 && ++b == NS) { b = 0; ph ^= 1; }
      bool done = false;
      if (left == 0) {
        const unsigned long long u = next_u;
        if (lane == 0) {   // consumed when this run ends
          // every CTA fetches once per run it starts plus once more (the ticket that stops
          // it): the launch's last fetch is number ntickets + G, after which no CTA touches
          // the counter again -- that fetch re-zeroes it for the next launch
          const unsigned long long old = atomicAdd(&A.ticket[0], 1ull);
          if (old == (unsigned long long)ntickets + (unsigned long long)G - 1ull) A.ticket[0] = 0;
          next_u = G + old;
        }
        next_u = __shfl_sync(0xffffffffu, next_u, 0);
        int t;
        if (u >= (unsigned long long)ntickets) {
          done = true;
          t = 0;
        } else if (u < (unsigned long long)nrun) {
          t = (int)u * run;
          left = run;
        } else {
          t = head + (int)(u - nrun);
          left = 1;
        }
        s = t / tps;
        tile = t - s * tps;
        t_id = t;
      }
      int32_t* hdr = reinterpret_cast<int32_t*>(metas + m * meta);
      if (done) {                                      // no tiles left: a stop entry for the compute warps
        if (k >= NS) mbar_wait(&empty[b], ph ^ 1);
        if (lane == 0) {
          hdr[0] = -1;
          mbar_arrive_tx(&full[b], 0);
        }
        break;
      }
      const int this_id = t_id, this_tile = tile;
      const int cs = s;
      --left;
      ++t_id;
      if (++tile == tps) { tile = 0; ++s; }
      const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)cs * P.desc_stride);
      const int32_t* prm = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(d) + kDescHeader);
      if (cs != loaded_s) {                            // the sample's descriptor, once per sample
        s_skip = d->skip != 0;
        S = src_rows_of(P, A, d, cs);
        top = prm[0]; ch = prm[2];
        loaded_s = cs;
      }
      const int r0 = this_tile * Rt, R = min(Rt, P.out_h - r0);
      const bool live = !s_skip && R > 0;
      if (this_tile == 0 && lane < A.sc.n_fields) {    // the batch's scalar fields, once per sample
        const int64_t i = A.sc.idx[cs];
        A.sc.outs[lane][cs] = A.sc.cols[lane][i];
      }
      int newxt = 0, ncopy = 0;
      bool per_row = false;
      const uint8_t* src0 = nullptr;                   // lane j: global address of slot j's first byte
      uint32_t tx = 0, my_sz = 0, my_base_out = 0;
      int ra = 0, rb = 0, ya_out = 0, yb_out = 0, wy_out = 0;
      if (live) {
        const int sh = S.sh;
        if (cs != cur_s) {   // a CTA's tiles of one sample are consecutive: its column range once per sample
          const int lft = prm[1], cwd = prm[3];
          if (affine) {
            bx0 = back_x(P, prm, 0);
            bxs = back_x(P, prm, 1) - bx0;
            by0 = back_y(P, prm, 0);
          }
          const int xa = affine ? bx0 : back_x(P, prm, 0), xb = affine ? bx0 + bxs * (OW - 1) : back_x(P, prm, OW - 1);
          int a0, a1, aw, b0, b1, bw;   // the composed maps are monotone: the end columns span the range
          lin_axis(min(xa, xb), P.canvas_w, cwd, P.lin32, P.linx_magic, a0, a1, aw);
          lin_axis(max(xa, xb), P.canvas_w, cwd, P.lin32, P.linx_magic, b0, b1, bw);
          col_lo = (lft + a0) >> sh;
          const int col_hi = (lft + b1) >> sh;
          span_bytes = col_hi >= col_lo ? (col_hi - col_lo + 1) * C : 0;
          // a row stride that is a multiple of 4 gives every staged row of the sample the
          // same byte phase mod 4 (the stage keeps the global phase mod 16): the column
          // table then carries it, and row offsets are word aligned
          aligned = (S.rstride & 3) == 0;
          cur_s = cs;
          newxt = 1;
          held_e = held_o = kCwNone;
        }
        int ya = 0, yb = 0, wy = 0;
        if (lane < R) {
          int y0, y1;
          lin_axis(affine ? by0 + r0 + lane : back_y(P, prm, r0 + lane), P.canvas_h, ch, P.lin32, P.liny_magic, y0, y1, wy);
          ya = (top + y0) >> sh;
          yb = (top + y1) >> sh;
        }
        // rows [lo, hi] are contiguous and at most nslot of them (host bound,
        // engine.cpp plan_compile: cw_slots)
        const int lo = __shfl_sync(0xffffffffu, ya, 0), hi = __shfl_sync(0xffffffffu, yb, R - 1);
        ncopy = span_bytes > 0 ? max(0, min(min(hi - lo + 1, nslot), S.rows - lo)) : 0;
        const uint32_t rstr = (uint32_t)S.rstride;
        // one copy per row when the row stride exceeds kCwPerRowNum / kCwPerRowDen x the window
        per_row = ncopy > 1 && (uint64_t)kCwPerRowDen * rstr > (uint64_t)kCwPerRowNum * (uint64_t)(span_bytes + 16);
        const uintptr_t a = reinterpret_cast<uintptr_t>(S.base + (int64_t)(lo + lane) * S.rstride + (int64_t)col_lo * C);
        uint32_t my_base;                              // stage offset of slot `lane`'s column col_lo
        if (per_row) {
          const uintptr_t al = a & ~(uintptr_t)15;
          my_base = (uint32_t)lane * span_pad + (uint32_t)(a - al);
          my_sz = lane < ncopy ? (uint32_t)((a - al + span_bytes + 15) & ~(uintptr_t)15) : 0u;
          src0 = reinterpret_cast<const uint8_t*>(al);
          tx = __reduce_add_sync(0xffffffffu, my_sz);
        } else {
          const uintptr_t a0 = reinterpret_cast<uintptr_t>(S.base + (int64_t)lo * S.rstride + (int64_t)col_lo * C);
          const uintptr_t al = a0 & ~(uintptr_t)15;
          const uint32_t base0 = (uint32_t)(a0 - al);
          my_base = base0 + (uint32_t)lane * rstr;
          if (ncopy > 0) tx = (uint32_t)((base0 + (uint64_t)(ncopy - 1) * rstr + span_bytes + 15) & ~(uint64_t)15);
          src0 = reinterpret_cast<const uint8_t*>(al);
        }
        if (aligned) my_base &= ~3u;                   // the phase is in the column table
        ra = lane < R ? ya - lo : 0;
        rb = lane < R ? yb - lo : 0;
        my_base_out = my_base;
        ya_out = ya; yb_out = yb; wy_out = wy;
      }
      // the tile's source rows go out first (the compute warps' release of tile
      // k - NS's stage), the rest of its geometry is written while they are in
      // flight; the full barrier completes on the bytes AND the arrive below
      if (k >= NS) mbar_wait(&empty[b], ph ^ 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint8_t* srcbuf = stages + (size_t)b * sbytes;
      if (tx) {
        if (lane == 0) mbar_expect_tx(&full[b], tx);
        __syncwarp();
        if (per_row) {
          if (lane < ncopy) bulk_g2s(srcbuf + (size_t)lane * span_pad, src0, my_sz, &full[b]);
        } else if (lane == 0) {
          bulk_g2s(srcbuf, src0, tx, &full[b]);
        }
      }
      if (live) {
        const int sh = S.sh;
        if (newxt && lane == 0) {                      // a new sample: the parameters of its column taps
          int32_t* cp = reinterpret_cast<int32_t*>(metas + m * meta + 16);
          const uint32_t ph4 = aligned ? (uint32_t)((reinterpret_cast<uintptr_t>(S.base) + (uintptr_t)col_lo * C) & 3u) : 0u;
          reinterpret_cast<int4*>(cp)[0] = make_int4(prm[1], prm[3], affine ? bx0 : INT32_MIN, bxs);
          reinterpret_cast<int4*>(cp)[1] = make_int4(col_lo, (int)ph4, sh, cs);
        }
        uint4* taps = reinterpret_cast<uint4*>(metas + m * meta + tap_off);
        const int ya = ya_out, yb = yb_out, wy = wy_out;
        const uint32_t my_base = my_base_out;
        const uint32_t ba = __shfl_sync(0xffffffffu, my_base, ra), bb = __shfl_sync(0xffffffffu, my_base, rb);
        // the two taps are one even and one odd absolute row (yb == ya + 1), or one row twice (bottom /
        // top clamp, or subsampled rows): that row takes all the weight, the other parity none
        uint32_t be = 0, bo = 0, te = kCwFake, to = kCwFake, wo = 0;
        if (lane < R) {
          if (ya == yb) {
            be = bo = ba;
            if (ya & 1) { to = (uint32_t)ya; wo = 2048u; }
            else te = (uint32_t)ya;
          } else if (ya & 1) {
            bo = ba; be = bb; to = (uint32_t)ya; te = (uint32_t)yb; wo = 2048u - (uint32_t)wy;
          } else {
            be = ba; bo = bb; te = (uint32_t)ya; to = (uint32_t)yb; wo = (uint32_t)wy;
          }
        }
        // new-row flags: a row is summed when it differs from the one the compute
        // warps hold for its parity (the last real row before it, this tile or the
        // sample's previous tiles in this CTA)
        const uint32_t me = __ballot_sync(0xffffffffu, te != kCwFake), mo = __ballot_sync(0xffffffffu, to != kCwFake);
        const uint32_t below = (1u << lane) - 1u, je = me & below, jo = mo & below;
        const uint32_t pe_l = __shfl_sync(0xffffffffu, te, je ? 31 - __clz(je) : 0);
        const uint32_t po_l = __shfl_sync(0xffffffffu, to, jo ? 31 - __clz(jo) : 0);
        const uint32_t pe = je ? pe_l : held_e, po = jo ? po_l : held_o;
        const uint32_t he_l = __shfl_sync(0xffffffffu, te, me ? 31 - __clz(me) : 0);
        const uint32_t ho_l = __shfl_sync(0xffffffffu, to, mo ? 31 - __clz(mo) : 0);
        if (me) held_e = he_l;
        if (mo) held_o = ho_l;
        if (lane < R) {
          const uint32_t fl = (te != kCwFake && te != pe ? 1u : 0u) | (to != kCwFake && to != po ? 2u : 0u);
          const uint32_t sb = stage0 + (uint32_t)b * (uint32_t)sbytes;
          taps[lane] = make_uint4(sb + be, sb + bo, fl, 4u * wo);
        }
      }
      if (lane == 0) {
        hdr[0] = this_id; hdr[1] = cs; hdr[2] = live ? 1 : 0; hdr[3] = newxt | (aligned ? 2 : 0);
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[b])) : "memory");
    }
    return;
  }

  // ---- compute warps
  const OutT* lut = reinterpret_cast<const OutT*>(smem);
  if constexpr (kMode == CW_LUT) {
    const uint4* g = reinterpret_cast<const uint4*>(A.lut);
    uint4* l4 = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < C * 256 * (int)sizeof(OutT) / 16; i += ncw * 32) l4[i] = g[i];
    asm volatile("bar.sync 1, %0;" ::"r"(ncw * 32) : "memory");   // compute warps only
  }
  const int pr = tid, npair = P.cw_npair;
  const bool act = pr < npair;
  const int ox0 = 2 * pr;
  const int nval = min(2, OW - ox0) * C;               // values this thread writes per row (6, or 3 at an odd edge)
  const size_t ostep = (size_t)OW * C;
  const bool vec = nval == 6 && (OW & 1) == 0;
  unsigned long long ab[3], bb[3];                     // affine map per value pair: channels (0,1) (2,0) (1,2)
  if constexpr (kMode == CW_AFFINE) {
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      ab[p] = reinterpret_cast<const unsigned long long*>(P.cw_pair_a)[p];   // distinct 64-bit pairs: no
      bb[p] = reinterpret_cast<const unsigned long long*>(P.cw_pair_b)[p];   // per-row re-pairing of 3 floats
    }
  }
  const unsigned long long magic2 = f2_pack(8388608.0f, 8388608.0f);
  // per owned column q: byte offset of its left tap in a staged row (word offset + shift
  // when the sample's rows are word aligned), tap weights, byte selectors
  uint32_t off[2] = {0, 0}, shf[2] = {0, 0}, wp[2] = {0, 0}, sel1[2] = {0, 0}, sel2[2] = {0, 0};
  uint32_t he[6], ho[6];                               // horizontal sums of the held even / odd source row
#pragma unroll
  for (int v = 0; v < 6; ++v) { he[v] = 0; ho[v] = 0; }
  bool al = false;
  for (int m = 0, b = 0, ph = 0;; m = m == NR - 1 ? 0 : m + 1) {
    mbar_wait(&full[b], ph);
    const int4 hd = *reinterpret_cast<const int4*>(metas + m * meta);   // ordered by the mbarrier wait (acquire)
    if (hd.x < 0) break;                               // the copy warp's stop entry
    if (hd.z && act) {
      const uint8_t* ent = metas + m * meta;
      if (hd.w & 1) {                                  // first tile of a sample: this thread's two column taps
        const int4 c0v = *reinterpret_cast<const int4*>(ent + 16), c1v = *reinterpret_cast<const int4*>(ent + 32);
        const int lft = c0v.x, cwd = c0v.y, bx0 = c0v.z, bxs = c0v.w, col_lo = c1v.x, sh = c1v.z;
        const uint32_t ph4 = (uint32_t)c1v.y;
        const int32_t* prm = bx0 == INT32_MIN   // crops / flips / resizes: the generic map from the descriptor
            ? reinterpret_cast<const int32_t*>(A.desc + (size_t)c1v.w * P.desc_stride + kDescHeader) : nullptr;
        al = (hd.w & 2) != 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int ox = min(ox0 + q, OW - 1);
          int x0, x1, wx;
          lin_axis(prm ? back_x(P, prm, ox) : bx0 + bxs * ox, P.canvas_w, cwd, P.lin32, P.linx_magic, x0, x1, wx);
          const int cc0 = (lft + x0) >> sh, cc1 = (lft + x1) >> sh;
          const uint32_t w1 = (uint32_t)wx, w0 = 2048u - w1;
          const uint32_t o = (uint32_t)((cc0 - col_lo) * C) + ph4;
          off[q] = al ? (o & ~3u) : o;
          shf[q] = (o & 3u) * 8u;
          wp[q] = w0 | w1 << 16;
          const bool same = cc1 == cc0;
          sel1[q] = same ? 0x1100u : 0x4130u;
          sel2[q] = same ? 0x0022u : 0x0052u;
        }
      }
      const int s = hd.y, tile = hd.x - s * tps;
      const int r0 = tile * Rt, R = min(Rt, P.out_h - r0);
      const uint4* taps = reinterpret_cast<const uint4*>(ent + tap_off);
      OutT* obase = reinterpret_cast<OutT*>(A.out) + ((size_t)s * P.out_h + r0) * ostep + (size_t)ox0 * C;
      auto rows = [&](auto kvec, auto kal) {
        constexpr bool kV = decltype(kvec)::value, kA = decltype(kal)::value;
        // the three channel sums of column q's two taps in the row at smem byte `a`
        auto sums = [&](uint32_t row, int q, uint32_t* h) {
          const uint32_t a = row + off[q];
          const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + (kA ? a : (a & ~3u)));
          const uint32_t sa = kA ? shf[q] : (a << 3);
          const uint32_t x = __funnelshift_r(w[0], w[1], sa), y = __funnelshift_r(w[1], w[2], sa);
          const uint32_t p1 = __byte_perm(x, y, sel1[q]), p2 = __byte_perm(x, y, sel2[q]);   // {a0 b0 a1 b1}, {a2 b2}
          h[0] = (uint32_t)dp2a_lo(wp[q], p1, 0);
          h[1] = (uint32_t)dp2a_hi(wp[q], p1, 0);
          h[2] = (uint32_t)dp2a_lo(wp[q], p2, 0);
        };
        OutT* o = obase;
#pragma unroll (kK1Unroll)
        for (int r = 0; r < R; ++r, o += ostep) {
          const uint4 tp = lds_v4(taps + r);             // one 128-bit load (the compiler splits a plain one)
          if (tp.z & 1u) { sums(tp.x, 0, he); sums(tp.x, 1, he + 3); }   // a new even source row
          if (tp.z & 2u) { sums(tp.y, 0, ho); sums(tp.y, 1, ho + 3); }   // a new odd source row
          const uint32_t wo4 = tp.w, we4 = 8192u - tp.w;
          uint32_t u[6];                               // 4 (w_e h_e + w_o h_o + 2^21): the value in bits 24..31
#pragma unroll
          for (int v = 0; v < 6; ++v) u[v] = he[v] * we4 + ho[v] * wo4 + (1u << 23);
          if constexpr (kMode == CW_AFFINE) {
            uint32_t pk[3];
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const unsigned long long x = f2_pack(__uint_as_float(u8_magic(u[2 * p])),
                                                   __uint_as_float(u8_magic(u[2 * p + 1])));
              pk[p] = cvt_pack2<OutT>(f2_fma(f2_sub(x, magic2), ab[p], bb[p]));
            }
            if constexpr (kV) {
              uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
              o32[0] = pk[0]; o32[1] = pk[1]; o32[2] = pk[2];
            } else {
#pragma unroll
              for (int v = 0; v < 6; ++v)
                if (v < nval) {
                  const uint16_t h = (uint16_t)(pk[v >> 1] >> (16 * (v & 1)));
                  memcpy(o + v, &h, 2);
                }
            }
          } else {
            OutT val[6];
#pragma unroll
            for (int v = 0; v < 6; ++v) {
              if constexpr (kMode == CW_LUT) val[v] = lut[(v % 3) * 256 + (u[v] >> 24)];
              else val[v] = (OutT)(u[v] >> 24);
            }
            if constexpr (kV && sizeof(OutT) <= 4) {
              using PT = typename std::conditional<sizeof(OutT) == 1, uint16_t,
                         typename std::conditional<sizeof(OutT) == 2, uint32_t, uint2>::type>::type;
              PT w3[3];
              memcpy(w3, val, sizeof w3);
              PT* op = reinterpret_cast<PT*>(o);
              op[0] = w3[0]; op[1] = w3[1]; op[2] = w3[2];
            } else {
#pragma unroll
              for (int v = 0; v < 6; ++v)
                if (v < nval) o[v] = val[v];
            }
          }
        }
      };
      if (vec) {
        if (al) rows(std::true_type{}, std::true_type{});
        else rows(std::true_type{}, std::false_type{});
      } else {
        if (al) rows(std::false_type{}, std::true_type{});
        else rows(std::false_type{}, std::false_type{});
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[b])) : "memory");
    if (++b == NS) { b = 0; ph ^= 1; }
  }
}

// ------------------------------------------------------------ K1 dispatch
// CTAs of a persistent kernel: SMs x resident CTAs per SM at this smem size
// (cached per kernel; the device is fixed for the process's loaders).
inline int persistent_ctas(const void* fn, int threads, int smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int64_t>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const int64_t key = (int64_t)threads << 32 | smem;
  auto it = cache.find({fn, key});
  if (it != cache.end()) return it->second;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
  const int n = std::max(1, sms) * std::max(1, per);
  cache[{fn, key}] = n;
  return n;
}
template <typename OutT, bool kRes, int kVal, int kC, bool kVec>
static int launch_img_t(const PlanDev& P, const LaunchArgs& A, cudaStream_t st) {
  if constexpr (kRes && kC == 3 && (kVal == VAL_LUT || kVal == VAL_COPY)) {
    if (P.cw) {   // the copy warp computes the geometry: no prologue launch
      auto k = image_cw_kernel<OutT, kVal == VAL_COPY ? CW_COPY : CW_LUT>;
      if constexpr (sizeof(OutT) == 2)
        if (P.cw_affine) k = image_cw_kernel<OutT, CW_AFFINE>;
      if (P.cw_smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, P.cw_smem);
      const int total = P.tiles_per_sample * A.count;
      const int threads = (P.cw_warps + 1) * 32;
      const int grid = std::min(total, persistent_ctas(reinterpret_cast<const void*>(k), threads, P.cw_smem));
      if (grid > 0) k<<<grid, threads, P.cw_smem, st>>>(P, A);
      return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
  }
  {   // prologue: per-sample geometry tables
    auto pk = sample_tables_kernel<kRes>;
    int tsm = (P.out_w + 3 * P.out_h) * 4;
    if (tsm > 48 * 1024) cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm);
    pk<<<A.count, kThreads, tsm, st>>>(P, A);
  }
  dim3 grid(P.tiles_per_sample, A.count);
  int smem = P.lay.total;
  auto k = image_kernel<OutT, kRes, kVal, kC, kVec>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<grid, kThreads, smem, st>>>(P, A);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <typename OutT, bool kRes, int kVal>
static int launch_img_c(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  switch (P.channels) {
    case 1: return vec ? launch_img_t<OutT, kRes, kVal, 1, true>(P, A, st) : launch_img_t<OutT, kRes, kVal, 1, false>(P, A, st);
    case 3: return vec ? launch_img_t<OutT, kRes, kVal, 3, true>(P, A, st) : launch_img_t<OutT, kRes, kVal, 3, false>(P, A, st);
    default: return launch_img_t<OutT, kRes, kVal, 0, false>(P, A, st);
  }
}

template <typename OutT, int kVal>
static int launch_img_r(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return P.src_kind == SRC_RESAMPLE ? launch_img_c<OutT, true, kVal>(P, A, st, vec)
                                    : launch_img_c<OutT, false, kVal>(P, A, st, vec);
}

template <typename OutT>
static int launch_img_typed(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  if constexpr (sizeof(OutT) == 1) {
    return launch_img_r<OutT, VAL_COPY>(P, A, st, vec);
  } else {
    if (P.value_mode == VAL_LUT) return launch_img_r<OutT, VAL_LUT>(P, A, st, vec);
    return launch_img_r<OutT, VAL_GENERIC>(P, A, st, vec);
  }
}

// one translation unit per output type (parallel build): kernels_img_*.cu
int launch_img_u8(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec);
int launch_img_f32(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec);
int launch_img_f16(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec);
int launch_img_bf16(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec);

}  // namespace bbx
