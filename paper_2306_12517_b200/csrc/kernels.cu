// sm_100a kernels of the bbox hot path.  See DESIGN.md §4 for the roofline of
// each kernel.  Nothing here is a dense contraction, so no tensor cores: the
// image kernel is an HBM-bound gather/expand, staged through shared memory so
// every global load is a 16-byte vector and every store a coalesced 16-byte
// vector of the channels-last (NHWC) output.
//
//   K1 image_kernel       Decode (RAW/SUBSAMPLE2/expanded-RLE canvas, zero pad)
//                         + RandomCrop/RandomFlip/Resize remaps + value ops
//                         (ToFloat/Normalize/per-channel/cast via exact LUT),
//                         or the bilinear RRC/CenterCrop decoders.
//                         Reference: pipeline.py:95-231, codecs.py:91-128.
//   K2 rle_expand_kernel  codecs.py:101-114 (RLE runs -> dense canvas), with
//                         the reference's error semantics as a status word.
//   K3 scalar_gather      loader.py:333-335 (label[b] = column[idx[b]]).
//   K3' array_kernel      ArrayRead (pipeline.py:128-129) + chain.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "bbx_internal.h"

namespace bbx {

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Output-to-input coordinate through the remaps, applied last-to-first.
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
__device__ __forceinline__ void lin_axis(int o, int out_n, int in_n, int& i0, int& i1, int& w1) {
  int64_t num = (int64_t)(2 * o + 1) * in_n - out_n, den = 2 * (int64_t)out_n;
  if (num <= 0) { i0 = 0; i1 = 0; w1 = 0; return; }
  int64_t q = num / den, r = num - q * den;
  if (q >= in_n - 1) { i0 = in_n - 1; i1 = in_n - 1; w1 = 0; return; }
  i0 = (int)q; i1 = (int)q + 1; w1 = (int)((r * 2048 + den / 2) / den);
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
  for (int i = 0; i < P.n_vops; ++i) {
    int kind = P.vop_kind[i];
    if (kind == BBX_OP_NORMALIZE) v = __fdiv_rn(__fsub_rn(v, P.vop_mean[i][0]), P.vop_std[i][0]);
    else if (kind == BBX_OP_NORMALIZE_PC) v = __fdiv_rn(__fsub_rn(v, P.vop_mean[i][k]), P.vop_std[i][k]);
  }
  return v;
}

template <typename T> __device__ __forceinline__ T cvt_out(float v);
template <> __device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <> __device__ __forceinline__ __half cvt_out<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ uint8_t cvt_out<uint8_t>(float v) { return (uint8_t)v; }

// Shared-memory layout of the image kernel (must match image_smem_bytes()).
struct ImgSmem {
  int etab_n;       // out_w * C entries
  int lut_bytes;
  int n_slots;      // staged source rows
  int span_pad;     // bytes per staged row
};

__host__ __device__ inline int align_up(int v, int a) { return (v + a - 1) / a * a; }

__host__ __device__ inline ImgSmem img_layout(const PlanDev& P, int out_size) {
  ImgSmem L;
  L.etab_n = P.out_w * P.out_c;
  L.lut_bytes = P.value_mode == VAL_LUT ? P.channels * 256 * out_size : 0;
  L.n_slots = P.rows_per_tile * (P.src_kind == SRC_RESAMPLE ? 2 : 1);
  // widest staged source row: the image row (<= canvas width for Decode,
  // <= max width for the resample decoders) plus 16 B of alignment slack.
  L.span_pad = align_up(P.src_row_w * P.channels, 16) + 32;
  return L;
}

// --------------------------------------------------------------------- K1
// grid = (tiles_per_sample, count); CTA = 256 threads = 8 warps.
// Phase A: per-column index tables + LUT into smem; per-row source addresses.
// Phase B: 16-byte vector copies of every needed source row segment into smem.
// Phase C: warp-per-output-row expansion, 16-byte coalesced NHWC stores.
template <typename OutT, bool kResample, int kVal, bool kVec>
__global__ void __launch_bounds__(kThreads, 4) image_kernel(const PlanDev P, const LaunchArgs A) {
  constexpr int V = kVec ? (16 / (int)sizeof(OutT)) : 1;
  const int s = blockIdx.y;
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  const int32_t* prm = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(d) + kDescHeader);
  if (d->skip) return;
  const int C = P.channels;
  const int r0 = blockIdx.x * P.rows_per_tile;
  const int R = min(P.rows_per_tile, P.out_h - r0);
  if (R <= 0) return;
  const int OW = P.out_w;
  const int rowlen = OW * C;
  const int h = d->h, w = d->w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const uint8_t* base;
  int sh;
  int64_t rstride;
  if (d->codec == CODEC_RLE) {
    base = A.scratch + (size_t)s * P.scratch_bytes; sh = 0; rstride = (int64_t)w * C;
  } else {
    base = A.payload + d->src; sh = d->codec == CODEC_SUB2 ? 1 : 0;
    rstride = (int64_t)(sh ? (w + 1) >> 1 : w) * C;
  }

  extern __shared__ __align__(16) uint8_t smem[];
  const ImgSmem L = img_layout(P, (int)sizeof(OutT));
  uint32_t* etab0 = reinterpret_cast<uint32_t*>(smem);
  uint32_t* etab1 = etab0 + L.etab_n;                       // resample only
  uint8_t* p = smem + (size_t)L.etab_n * 4 * (kResample ? 2 : 1);
  OutT* lut = reinterpret_cast<OutT*>(p);
  p += align_up(L.lut_bytes, 16);
  int* slot_off = reinterpret_cast<int*>(p);                 // per staged row: smem byte offset, -1 = zero row
  int* slot_src = slot_off + L.n_slots;                       // per staged row: source row index
  int* row_wy = slot_src + L.n_slots;                         // resample: wy per output row
  p += align_up(L.n_slots * 8 + P.rows_per_tile * 4, 16);
  uint8_t* rows = p;

  // ---- column range (composition of monotone maps: extremes at the ends)
  int col_lo, col_hi;   // inclusive, in source-row element columns (after >> sh)
  int top = 0, left = 0, ch = 0, cw = 0;
  if (kResample) {
    top = prm[0]; left = prm[1]; ch = prm[2]; cw = prm[3];
    int xa = back_x(P, prm, 0), xb = back_x(P, prm, OW - 1);
    int lo = min(xa, xb), hi = max(xa, xb), a0, a1, aw, b0, b1, bw;
    lin_axis(lo, P.canvas_w, cw, a0, a1, aw);
    lin_axis(hi, P.canvas_w, cw, b0, b1, bw);
    col_lo = (left + a0) >> sh; col_hi = (left + b1) >> sh;
  } else {
    int xa = back_x(P, prm, 0), xb = back_x(P, prm, OW - 1);
    int lo = min(xa, xb), hi = min(max(xa, xb), w - 1);
    col_lo = lo >> sh; col_hi = hi >> sh;   // col_lo > col_hi: every column is padding
  }
  const int64_t span_bytes = col_hi >= col_lo ? (int64_t)(col_hi - col_lo + 1) * C : 0;

  // ---- phase A: tables
  if (kVal == VAL_LUT) {
    const OutT* g = reinterpret_cast<const OutT*>(A.lut);
    for (int i = tid; i < C * 256; i += kThreads) lut[i] = g[i];
  }
  for (int ox = tid; ox < OW; ox += kThreads) {
    if (kResample) {
      int cx = back_x(P, prm, ox), x0, x1, wx;
      lin_axis(cx, P.canvas_w, cw, x0, x1, wx);
      int o0 = (((left + x0) >> sh) - col_lo) * C, o1 = (((left + x1) >> sh) - col_lo) * C;
      for (int k = 0; k < C; ++k) {
        etab0[ox * C + k] = (uint32_t)(o0 + k) | ((uint32_t)k << 16);
        etab1[ox * C + k] = (uint32_t)(o1 + k) | ((uint32_t)wx << 16);
      }
    } else {
      int cx = back_x(P, prm, ox);
      bool valid = cx < w;
      int o = ((cx >> sh) - col_lo) * C;
      for (int k = 0; k < C; ++k)
        etab0[ox * C + k] = valid ? ((uint32_t)(o + k) | ((uint32_t)k << 16)) : (0xFFFFu | ((uint32_t)k << 16));
    }
  }
  // per staged row: global source address (thread-per-row)
  for (int r = tid; r < R; r += kThreads) {
    if (kResample) {
      int cy = back_y(P, prm, r0 + r), y0, y1, wy;
      lin_axis(cy, P.canvas_h, ch, y0, y1, wy);
      row_wy[r] = wy;
      slot_src[2 * r] = (top + y0) >> sh;
      slot_src[2 * r + 1] = (top + y1) >> sh;
    } else {
      int cy = back_y(P, prm, r0 + r);
      slot_src[r] = (cy < h && span_bytes > 0) ? (cy >> sh) : -1;
    }
  }
  __syncthreads();

  // ---- phase B: 16-byte vector copies of the source row segments (warp per row)
  const int n_slots = kResample ? 2 * R : R;
  for (int j = warp; j < n_slots; j += kThreads / 32) {
    int srow = slot_src[j];
    uint8_t* dst = rows + (size_t)j * L.span_pad;
    if (srow < 0) { if (lane == 0) slot_off[j] = -1; continue; }
    const uint8_t* src = base + (int64_t)srow * rstride + (int64_t)col_lo * C;
    uintptr_t a = reinterpret_cast<uintptr_t>(src);
    uintptr_t a0 = a & ~(uintptr_t)15;
    int shift = (int)(a - a0);
    int n16 = (int)((shift + span_bytes + 15) >> 4);
    const uint8_t* s0 = reinterpret_cast<const uint8_t*>(a0);
    for (int c = lane; c < n16; c += 32)
      *reinterpret_cast<uint4*>(dst + 16 * c) = ld_nc_v4(s0 + 16 * c);
    if (lane == 0) slot_off[j] = j * L.span_pad + shift;
  }
  __syncthreads();

  // ---- phase C: expand (warp per output row)
  OutT* out = reinterpret_cast<OutT*>(A.out) + ((size_t)s * P.out_h + r0) * rowlen;
  for (int r = warp; r < R; r += kThreads / 32) {
    const uint8_t* row0;
    const uint8_t* row1 = nullptr;
    int wy = 0;
    bool rv;
    if (kResample) {
      row0 = smem + slot_off[2 * r]; row1 = smem + slot_off[2 * r + 1]; wy = row_wy[r]; rv = true;
    } else {
      rv = slot_off[r] >= 0;
      row0 = smem + (rv ? slot_off[r] : 0);
    }
    OutT* orow = out + (size_t)r * rowlen;
    for (int q = lane * V; q < rowlen; q += 32 * V) {
      union { OutT v[V]; uint4 u; } pk;
      OutT* vals = pk.v;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        uint32_t e = etab0[q + i];
        int off = (int)(e & 0xFFFFu), k = (int)(e >> 16);
        uint32_t b;
        if (kResample) {
          uint32_t e1 = etab1[q + i];
          int off1 = (int)(e1 & 0xFFFFu), wx = (int)(e1 >> 16);
          k = (int)((e >> 16) & 0xFFFFu);
          uint32_t t0 = (uint32_t)(2048 - wx) * row0[off] + (uint32_t)wx * row0[off1];
          uint32_t t1 = (uint32_t)(2048 - wx) * row1[off] + (uint32_t)wx * row1[off1];
          b = ((uint32_t)(2048 - wy) * t0 + (uint32_t)wy * t1 + (1u << 21)) >> 22;
        } else {
          b = (rv && off != 0xFFFF) ? row0[off] : 0u;
        }
        if (kVal == VAL_LUT) vals[i] = lut[k * 256 + b];
        else if (kVal == VAL_COPY) vals[i] = (OutT)b;
        else vals[i] = cvt_out<OutT>(apply_vops(P, (float)b, k));
      }
      if (kVec) {
        *reinterpret_cast<uint4*>(orow + q) = pk.u;
      } else {
        orow[q] = vals[0];
      }
    }
  }
}

// --------------------------------------------------------------------- K2
// One CTA per RLE sample.  Runs are processed in chunks of 1024: a block scan
// turns counts into start positions, then every thread expands a contiguous
// share of the chunk's output (one binary search, then a walk).  Error rules
// of codecs.py:101-114: any zero count or a prefix sum past n -> "past";
// otherwise a total != n -> "sum to".
constexpr int kRleRunsPerThread = 4;
constexpr int kRleChunk = kThreads * kRleRunsPerThread;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* warp_tot, uint64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < kThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kThreads / 32) warp_tot[lane] = t;   // inclusive
  }
  __syncthreads();
  uint64_t before = warp ? warp_tot[warp - 1] : 0;
  total = warp_tot[kThreads / 32 - 1];
  return before + x - v;
}

__global__ void __launch_bounds__(kThreads) rle_expand_kernel(const PlanDev P, const LaunchArgs A) {
  const int s = blockIdx.x;
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  if (d->skip || d->codec != CODEC_RLE) return;
  __shared__ uint64_t starts[kRleChunk + 1];
  __shared__ uint8_t vals[kRleChunk];
  __shared__ uint64_t warp_tot[kThreads / 32];
  __shared__ int s_err;
  const uint8_t* pay = A.payload + d->src;
  const int64_t nruns = d->len / 5;
  const uint64_t n = (uint64_t)d->h * d->w * d->c;
  uint8_t* out = A.scratch + (size_t)s * P.scratch_bytes;
  if (threadIdx.x == 0) s_err = 0;
  uint64_t carry = 0;
  __syncthreads();
  for (int64_t cb = 0; cb < nruns; cb += kRleChunk) {
    uint32_t cnt[kRleRunsPerThread];
    uint64_t tsum = 0;
    bool zero = false;
#pragma unroll
    for (int j = 0; j < kRleRunsPerThread; ++j) {
      int64_t ri = cb + threadIdx.x * kRleRunsPerThread + j;
      cnt[j] = 0;
      if (ri < nruns) {
        const uint8_t* q = pay + ri * 5;
        cnt[j] = (uint32_t)q[0] | (uint32_t)q[1] << 8 | (uint32_t)q[2] << 16 | (uint32_t)q[3] << 24;
        vals[threadIdx.x * kRleRunsPerThread + j] = q[4];
        zero |= cnt[j] == 0;
      }
      tsum += cnt[j];
    }
    if (zero) s_err = 1;
    uint64_t total;
    uint64_t st = carry + block_excl_scan(tsum, warp_tot, total);
#pragma unroll
    for (int j = 0; j < kRleRunsPerThread; ++j) {
      starts[threadIdx.x * kRleRunsPerThread + j] = st;
      st += cnt[j];
    }
    const int in_chunk = (int)(nruns - cb < (int64_t)kRleChunk ? nruns - cb : (int64_t)kRleChunk);
    if (threadIdx.x == 0) starts[in_chunk] = carry + total;
    __syncthreads();
    if (carry + total > n) s_err = 1;
    __syncthreads();
    if (!s_err) {
      // expand [carry, carry+total): thread t takes a contiguous share
      uint64_t per = (total + kThreads - 1) / kThreads;
      uint64_t p0 = carry + per * threadIdx.x, p1 = min(carry + total, p0 + per);
      if (p0 < p1) {
        int lo = 0, hi = in_chunk - 1;   // largest j with starts[j] <= p0
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (starts[mid] <= p0) lo = mid; else hi = mid - 1;
        }
        int j = lo;
        for (uint64_t pos = p0; pos < p1; ++pos) {
          while (starts[j + 1] <= pos) ++j;
          out[pos] = vals[j];
        }
      }
    }
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    SampleStatus stt{0, 0, 0};
    if (s_err) { stt.kind = 1; stt.value = (int64_t)n; }
    else if (carry != n) { stt.kind = 2; stt.value = (int64_t)carry; }
    A.status[s] = stt;
  }
}

// --------------------------------------------------------------------- K3
__global__ void scalar_gather_kernel(const ScalarArgs S) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= S.count) return;
  int64_t i = S.idx[b];
  for (int f = 0; f < S.n_fields; ++f) S.outs[f][b] = S.cols[f][i];
}

// FIXED_ARRAY chains: element-wise gather (+ 3-D remaps) + value ops.
template <bool kDirect, typename OutT>
__global__ void __launch_bounds__(kThreads) array_kernel(const PlanDev P, const LaunchArgs A) {
  const int s = blockIdx.y;
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  if (d->skip) return;
  const int32_t* prm = reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(d) + kDescHeader);
  const uint8_t* src = A.payload + d->src;
  const int E = P.src_elem;
  const int64_t n = P.out_sample_elems;
  const int C = P.out_c, OW = P.out_w;
  uint8_t* outb = reinterpret_cast<uint8_t*>(A.out);
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kThreads) {
    int64_t si = e;
    int k = 0;
    if (P.has_remaps_3d) {
      int64_t y = e / ((int64_t)OW * C);
      int x = (int)((e / C) % OW);
      k = (int)(e % C);
      int sy = back_y(P, prm, (int)y), sx = back_x(P, prm, x);
      si = ((int64_t)sy * P.canvas_w + sx) * P.channels + k;
    } else if (C > 1) {
      k = (int)(e % C);
    }
    const uint8_t* sp = src + si * E;
    if (kDirect) {
      float v = apply_vops(P, to_f32(sp, P.src_dtype), k);
      reinterpret_cast<OutT*>(outb)[(size_t)s * n + e] = cvt_out<OutT>(v);
    } else {
      uint8_t* dp = outb + ((size_t)s * n + e) * E;
      for (int b = 0; b < E; ++b) dp[b] = sp[b];
    }
  }
}

// ------------------------------------------------------------------ launch

int image_smem_bytes(const PlanDev& P) {
  int osz = P.out_dtype == BBX_U8 ? 1 : (P.out_dtype == BBX_F32 ? 4 : 2);
  ImgSmem L = img_layout(P, osz);
  int bytes = L.etab_n * 4 * (P.src_kind == SRC_RESAMPLE ? 2 : 1);
  bytes += align_up(L.lut_bytes, 16);
  bytes += align_up(L.n_slots * 8 + P.rows_per_tile * 4, 16);
  bytes += L.n_slots * L.span_pad;
  return bytes;
}

template <typename OutT, bool kRes, int kVal>
static int launch_img_t(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  dim3 grid(P.tiles_per_sample, A.count);
  int smem = image_smem_bytes(P);
  if (vec) {
    auto k = image_kernel<OutT, kRes, kVal, true>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, kThreads, smem, st>>>(P, A);
  } else {
    auto k = image_kernel<OutT, kRes, kVal, false>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, kThreads, smem, st>>>(P, A);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <typename OutT, int kVal>
static int launch_img_r(const PlanDev& P, const LaunchArgs& A, cudaStream_t st, bool vec) {
  return P.src_kind == SRC_RESAMPLE ? launch_img_t<OutT, true, kVal>(P, A, st, vec)
                                    : launch_img_t<OutT, false, kVal>(P, A, st, vec);
}

int launch_image(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int osz = P.out_dtype == BBX_U8 ? 1 : (P.out_dtype == BBX_F32 ? 4 : 2);
  bool vec = ((int64_t)P.out_w * P.out_c * osz) % 16 == 0 &&
             (reinterpret_cast<uintptr_t>(A.out) & 15) == 0;
  switch (P.out_dtype) {
    case BBX_U8:
      return launch_img_r<uint8_t, VAL_COPY>(P, A, st, vec);
    case BBX_F32:
      return P.value_mode == VAL_LUT ? launch_img_r<float, VAL_LUT>(P, A, st, vec)
                                     : launch_img_r<float, VAL_DIRECT>(P, A, st, vec);
    case BBX_F16:
      return P.value_mode == VAL_LUT ? launch_img_r<__half, VAL_LUT>(P, A, st, vec)
                                     : launch_img_r<__half, VAL_DIRECT>(P, A, st, vec);
    case BBX_BF16:
      return P.value_mode == VAL_LUT ? launch_img_r<__nv_bfloat16, VAL_LUT>(P, A, st, vec)
                                     : launch_img_r<__nv_bfloat16, VAL_DIRECT>(P, A, st, vec);
  }
  return -1;
}

int launch_rle_expand(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  rle_expand_kernel<<<A.count, kThreads, 0, (cudaStream_t)stream>>>(P, A);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_array(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t tiles = (P.out_sample_elems + kThreads * 8 - 1) / (kThreads * 8);
  if (tiles > 65535) tiles = 65535;
  dim3 grid((unsigned)tiles, A.count);
  if (P.value_mode == VAL_COPY) {
    array_kernel<false, float><<<grid, kThreads, 0, st>>>(P, A);
  } else {
    switch (P.out_dtype) {
      case BBX_F32: array_kernel<true, float><<<grid, kThreads, 0, st>>>(P, A); break;
      case BBX_F16: array_kernel<true, __half><<<grid, kThreads, 0, st>>>(P, A); break;
      case BBX_BF16: array_kernel<true, __nv_bfloat16><<<grid, kThreads, 0, st>>>(P, A); break;
      default: return -1;
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_scalar_gather(const ScalarArgs& S, void* stream) {
  if (S.count <= 0 || S.n_fields == 0) return 0;
  scalar_gather_kernel<<<(S.count + 255) / 256, 256, 0, (cudaStream_t)stream>>>(S);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace bbx
