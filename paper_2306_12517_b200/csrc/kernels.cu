// sm_100a kernels of the bbox hot path besides K1 (image_kernel.cuh):
//   K2 rle_expand_kernel  codecs.py:101-114 (RLE runs -> dense canvas), with
//                         the reference's error semantics as a status word.
//   K3 scalar_gather      loader.py:333-335 (label[b] = column[idx[b]]).
//   K3' array_kernel      ArrayRead (pipeline.py:128-129) + chain.
#include "image_kernel.cuh"

namespace bbx {

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
// FIXED_ARRAY chains without remaps or value ops (ArrayRead alone, pipeline.py:
// 128-129): a straight copy of each sample's payload into its output row,
// 16-byte aligned stores; the source is read as aligned 16-byte chunks and
// realigned with funnel shifts (its misalignment is uniform per sample).
template <int kQ>
__device__ __forceinline__ uint4 realign(const uint4 a, const uint4 b, uint32_t r) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  return make_uint4(__funnelshift_r(w[kQ], w[kQ + 1], r), __funnelshift_r(w[kQ + 1], w[kQ + 2], r),
                    __funnelshift_r(w[kQ + 2], w[kQ + 3], r), __funnelshift_r(w[kQ + 3], w[kQ + 4], r));
}
__global__ void __launch_bounds__(kThreads) array_copy_kernel(const PlanDev P, const LaunchArgs A) {
  const int s = blockIdx.y;
  const SampleDesc* d = reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * P.desc_stride);
  if (d->skip) return;
  const int64_t len = P.out_sample_elems * P.src_elem;
  const uint8_t* src = A.payload + d->src;
  uint8_t* dst = reinterpret_cast<uint8_t*>(A.out) + (size_t)s * len;
  const int64_t al = (16 - (int64_t)(reinterpret_cast<uintptr_t>(dst) & 15)) & 15, head = al < len ? al : len;
  const int64_t nchunk = (len - head) >> 4;
  const int64_t tail0 = head + nchunk * 16;
  const int64_t t0 = (int64_t)blockIdx.x * kThreads + threadIdx.x, step = (int64_t)gridDim.x * kThreads;
  if (t0 < head) dst[t0] = src[t0];
  if (t0 < len - tail0) dst[tail0 + t0] = src[tail0 + t0];
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(src + head);
  const int sh = (int)(a0 & 15);
  const uint4* s4 = reinterpret_cast<const uint4*>(a0 - sh);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  const uint32_t r = (uint32_t)(sh & 3) * 8;
  switch (sh >> 2) {   // uniform per sample
#define BBX_COPY_CASE(Q)                                                                   \
    case Q:                                                                               \
      for (int64_t c = t0; c < nchunk; c += step) {                                       \
        const uint4 lo = ld_nc_v4(s4 + c);                                                \
        const uint4 hi = sh ? ld_nc_v4(s4 + c + 1) : lo;                                  \
        d4[c] = realign<Q>(lo, hi, r);                                                    \
      }                                                                                   \
      break;
    BBX_COPY_CASE(0) BBX_COPY_CASE(1) BBX_COPY_CASE(2) BBX_COPY_CASE(3)
#undef BBX_COPY_CASE
  }
}

// ------------------------------------------------------------------ launch

int image_smem_bytes(const PlanDev& P) { return img_layout(P).total; }
SmemLayout img_layout_host(const PlanDev& P) { return img_layout(P); }
int image_tab_stride(const PlanDev& P) { return tab_stride(P); }
int cw_smem_host(const PlanDev& P) { return cw_smem_bytes(P); }

int launch_image(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int osz = P.out_dtype == BBX_U8 ? 1 : (P.out_dtype == BBX_F32 ? 4 : 2);
  int V = 16 / osz;
  bool vec = P.out_w % V == 0 && (reinterpret_cast<uintptr_t>(A.out) & 15) == 0;
  switch (P.out_dtype) {
    case BBX_U8: return launch_img_u8(P, A, st, vec);
    case BBX_F32: return launch_img_f32(P, A, st, vec);
    case BBX_F16: return launch_img_f16(P, A, st, vec);
    case BBX_BF16: return launch_img_bf16(P, A, st, vec);
  }
  return -1;
}

int launch_rle_expand(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  rle_expand_kernel<<<A.count, kThreads, 0, (cudaStream_t)stream>>>(P, A);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Zero-copy gather: the batch's payload rows, read by the SMs straight from the
// pinned + mapped host heap over PCIe (the CPU touches none of the bytes: one host
// DRAM read per byte, against three for gather -> pinned slot -> DMA), into the
// slot's device payload region, which K1 then reads as a staged batch.  CTA per
// copy; a warp per 496-byte segment of a row: 32 lanes load the 32 aligned
// 16-byte chunks that cover it and lanes 0..30 each assemble one unaligned
// 16-byte output chunk from their chunk and the next lane's (shuffle + funnel).
__global__ void __launch_bounds__(256) host_gather_kernel(const uint8_t* __restrict__ heap, uint64_t heap_bytes,
                                                          uint8_t* __restrict__ slot,
                                                          const GatherCopy* __restrict__ copies) {
  const GatherCopy c = copies[blockIdx.x];
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr uint32_t kSeg = 31 * 16;
  const uint32_t spr = (c.row_bytes + kSeg - 1) / kSeg;
  for (uint32_t sg = threadIdx.x >> 5; sg < c.rows * spr; sg += nw) {
    const uint32_t r = sg / spr, q = sg - r * spr;
    const uint64_t row = c.src + (uint64_t)r * c.src_stride, s = row + (uint64_t)q * kSeg;
    const uint64_t end = min(row + c.row_bytes, heap_bytes);          // loads never pass the row's last chunk
    const uint64_t al = s & ~15ull, at = al + 16ull * (uint64_t)lane;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (at < end) v = *reinterpret_cast<const uint4*>(heap + at);
    uint4 nx;
    nx.x = __shfl_down_sync(0xffffffffu, v.x, 1);
    nx.y = __shfl_down_sync(0xffffffffu, v.y, 1);
    nx.z = __shfl_down_sync(0xffffffffu, v.z, 1);
    nx.w = __shfl_down_sync(0xffffffffu, v.w, 1);
    const uint32_t o = q * kSeg + 16u * (uint32_t)lane;               // output byte of this lane's chunk in the row
    if (lane == 31 || o >= c.row_bytes) continue;
    // bytes [sh, sh + 16) of the 32 bytes (v, nx): whole words first, then the byte shift
    const uint32_t sh = (uint32_t)(s & 15);
    uint32_t w0 = v.x, w1 = v.y, w2 = v.z, w3 = v.w, w4 = nx.x, w5 = nx.y, w6 = nx.z, w7 = nx.w;
    if (sh & 8) { w0 = w2; w1 = w3; w2 = w4; w3 = w5; w4 = w6; w5 = w7; }
    if (sh & 4) { w0 = w1; w1 = w2; w2 = w3; w3 = w4; w4 = w5; }
    const uint32_t bs = (sh & 3) * 8;
    const uint4 out = make_uint4(__funnelshift_r(w0, w1, bs), __funnelshift_r(w1, w2, bs), __funnelshift_r(w2, w3, bs),
                                 __funnelshift_r(w3, w4, bs));
    *reinterpret_cast<uint4*>(slot + c.dst + (uint64_t)r * c.dst_stride + o) = out;
  }
}

int launch_host_gather(const uint8_t* heap, uint64_t heap_bytes, uint8_t* slot, const GatherCopy* copies, int n,
                       void* stream) {
  if (n <= 0) return 0;
  host_gather_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(heap, heap_bytes, slot, copies);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_array(const PlanDev& P, const LaunchArgs& A, void* stream) {
  if (A.count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t tiles = (P.out_sample_elems + kThreads * 8 - 1) / (kThreads * 8);
  if (tiles > 65535) tiles = 65535;
  dim3 grid((unsigned)tiles, A.count);
  if (P.value_mode == VAL_COPY && !P.has_remaps_3d) {
    const int64_t chunks = (P.out_sample_elems * P.src_elem + 15) / 16;
    dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>((chunks + kThreads * 4 - 1) / (kThreads * 4), 65535)),
           A.count);
    array_copy_kernel<<<g, kThreads, 0, st>>>(P, A);
  } else if (P.value_mode == VAL_COPY) {
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
