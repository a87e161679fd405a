// sm_100a JPEG decoder (codec id 3) — the decode stage of Decode /
// RandomResizedCrop / CenterCrop on JPEG samples.  See jpeg.h for the
// pipeline (J1 marker scan, J2 Huffman, J3 IDCT, J4 upsample + color) and
// DESIGN.md §4 for the roofline of each step.
//
// Numerics follow libjpeg-turbo's defaults (ISLOW IDCT, fancy upsampling,
// 16-bit fixed-point YCbCr->RGB), restated in oracle/jpeg_oracle.c and
// pinned bit-exact against Pillow; this file must agree with that oracle bit
// for bit.  All arithmetic is integer.
#include <cuda_runtime.h>

#include "bbx_internal.h"
#include "jpeg.h"

namespace bbx {

__constant__ uint8_t c_natural[80] = {   // zig-zag -> natural, + overrun guard (T.81 Fig. A.6)
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33,
    40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36,
    29, 22, 15, 23, 30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54,
    47, 55, 62, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63};

__device__ __forceinline__ const SampleDesc* sdesc(const JpegArgs& A, int s) {
  return reinterpret_cast<const SampleDesc*>(A.desc + (size_t)s * A.desc_stride);
}

// ------------------------------------------------------------------- J1
// Warp per sample.  Lanes read consecutive 16-byte chunks of the entropy-
// coded segment; a pair (0xFF, 0xD0..0xD7) is a restart marker (inside coded
// data 0xFF is always followed by 0x00).  A warp scan orders the markers:
// marker k ends interval k and interval k+1 starts two bytes later.
constexpr int kScanWarps = 4;

__global__ void __launch_bounds__(32 * kScanWarps) jpeg_scan_kernel(const JpegArgs A) {
  const int s = blockIdx.x * kScanWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (s >= A.count) return;
  const JpegDesc& J = A.jd[s];
  const uint32_t nint = J.n_int;
  if (nint == 0) return;
  const uint8_t* base = A.payload + sdesc(A, s)->src;
  const uint32_t lo = J.scan_off, hi = J.scan_end;
  uint32_t* st = A.istart + J.int_base;
  uint32_t* en = A.iend + J.int_base;
  if (lane == 0) st[0] = lo;
  const uintptr_t ab = reinterpret_cast<uintptr_t>(base);
  const uintptr_t a_lo = ab + lo, a_hi = ab + hi;
  uint32_t found = 0;
  bool seq_bad = false;
  for (uintptr_t c = a_lo & ~uintptr_t(15); c < a_hi; c += 512) {
    const uintptr_t my = c + (uintptr_t)lane * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (my < a_hi) v = *reinterpret_cast<const uint4*>(my);   // buffers carry >= 16 B of tail padding
    uint32_t nxt = __shfl_down_sync(0xffffffffu, v.x & 0xFF, 1);
    if (lane == 31) nxt = (my + 16 < a_hi) ? *reinterpret_cast<const uint8_t*>(my + 16) : 0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t b = (w[j >> 2] >> ((j & 3) * 8)) & 0xFF;
      const uint32_t n = j < 15 ? (w[(j + 1) >> 2] >> (((j + 1) & 3) * 8)) & 0xFF : nxt;
      const uintptr_t pos = my + j;
      if (b == 0xFF && (n & 0xF8) == 0xD0 && pos >= a_lo && pos + 1 < a_hi) mask |= 1u << j;
    }
    const uint32_t cnt = __popc(mask);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t k = found + incl - cnt;
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint32_t rel = (uint32_t)(my + j - ab);
      const uint32_t marker = (j < 15 ? (w[(j + 1) >> 2] >> (((j + 1) & 3) * 8)) : nxt) & 7;
      if (marker != (k & 7)) seq_bad = true;
      if (k + 1 < nint) { en[k] = rel; st[k + 1] = rel + 2; }
      ++k;
    }
    found += __shfl_sync(0xffffffffu, incl, 31);
  }
  seq_bad = __any_sync(0xffffffffu, seq_bad);
  if (lane == 0) {
    SampleStatus& S = A.status[s];
    S.kind = 0; S.value = 0;
    if (found != nint - 1) { S.kind = JST_MARKER_COUNT; S.value = found; }
    else if (seq_bad) S.kind = JST_MARKER_SEQ;
    else en[nint - 1] = hi;
  }
}

// ------------------------------------------------------------------- J2
// Thread per restart interval: the interval's MCUs are decoded serially (DC
// predictors restart at zero, T.81 F.2.1.3.1).  The bit reader keeps up to 64
// bits MSB-first; 0xFF00 is unstuffed on the fly and the first 0xFF followed
// by anything else ends the data (zero bits from there on, as libjpeg does).
constexpr int kHuffThreads = 128;

struct BitReader {
  uint64_t acc;
  int nb;
  const uint8_t* p;
  const uint8_t* pe;
  __device__ __forceinline__ void refill() {
    while (nb <= 56) {
      uint32_t b = 0;
      if (p < pe) {
        b = *p;
        if (b == 0xFF) {
          if (p + 1 < pe && p[1] == 0) p += 2;
          else { pe = p; b = 0; }
        } else {
          ++p;
        }
      }
      acc |= (uint64_t)b << (56 - nb);
      nb += 8;
    }
  }
  __device__ __forceinline__ int bits(int s) {   // 1 <= s <= 16, nb >= s
    const int v = (int)(acc >> (64 - s));
    acc <<= s;
    nb -= s;
    return v;
  }
};

__device__ __forceinline__ int huff_symbol(const JHuff* __restrict__ T, BitReader& br, bool& bad) {
  const uint32_t e = __ldg(&T->look[(uint32_t)(br.acc >> (64 - kJpegLook))]);
  int len, sym;
  if (e) {
    len = (int)(e >> 8);
    sym = (int)(e & 0xFF);
  } else {                                           // codes longer than the lookahead
    const uint32_t c16 = (uint32_t)(br.acc >> 48);
    len = kJpegLook + 1;
    while (len <= 16 && (int32_t)(c16 >> (16 - len)) > __ldg(&T->maxcode[len])) ++len;
    if (len > 16) { bad = true; len = 16; sym = 0; }
    else sym = __ldg(&T->vals[(c16 >> (16 - len)) + __ldg(&T->valoff[len])]);
  }
  br.acc <<= len;
  br.nb -= len;
  return sym;
}

__device__ __forceinline__ int extend(int v, int s) { return v < (1 << (s - 1)) ? v - (1 << s) + 1 : v; }

template <typename T>
__device__ __forceinline__ int find_sample(const T* prefix, int count, T t) {   // largest s: prefix[s] <= t
  int lo = 0, hi = count;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&prefix[mid]) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kHuffThreads) jpeg_huffman_kernel(const JpegArgs A) {
  __shared__ uint8_t nat[80];
  if (threadIdx.x < 80) nat[threadIdx.x] = c_natural[threadIdx.x];
  __syncthreads();
  const uint32_t t = blockIdx.x * kHuffThreads + threadIdx.x;
  if (t >= A.total_int) return;
  const int s = find_sample(A.int_prefix, A.count, t);
  if (A.status[s].kind != 0) return;                 // J1 rejected the marker layout
  const JpegDesc& J = A.jd[s];
  const uint32_t k = t - J.int_base;
  const uint8_t* base = A.payload + sdesc(A, s)->src;
  BitReader br{0, 0, base + A.istart[t], base + A.iend[t]};
  const uint32_t total = (uint32_t)J.mcus_x * J.mcus_y;
  const uint32_t m0 = k * J.restart, m1 = min(m0 + J.restart, total);
  const int ncomp = J.ncomp;
  int pred[3] = {0, 0, 0};
  bool bad = false;
  uint32_t mx = m0 % J.mcus_x, my = m0 / J.mcus_x;
  for (uint32_t m = m0; m < m1 && !bad; ++m) {
#pragma unroll
    for (int ci = 0; ci < 3; ++ci) {
      if (ci >= ncomp) break;
      const JComp& C = J.comp[ci];
      const JHuff* dct = A.huff + C.dc;
      const JHuff* act = A.huff + C.ac;
      for (int v = 0; v < C.v; ++v)
        for (int h = 0; h < C.h; ++h) {
          const size_t blk = J.blk_base + C.blk_off + (size_t)(my * C.v + v) * C.bw + (mx * C.h + h);
          int16_t* out = A.coef + blk * 64;
          uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
          for (int i = 0; i < 8; ++i) o4[i] = make_uint4(0, 0, 0, 0);
          if (br.nb < 32) br.refill();
          const int tdc = huff_symbol(dct, br, bad);
          int diff = 0;
          if (tdc) { if (br.nb < 16) br.refill(); diff = extend(br.bits(tdc), tdc); }
          pred[ci] += diff;
          out[0] = (int16_t)pred[ci];
          for (int kk = 1; kk < 64; ++kk) {
            if (br.nb < 32) br.refill();
            const int rs = huff_symbol(act, br, bad);
            const int run = rs >> 4, sz = rs & 15;
            if (sz) {
              kk += run;
              out[nat[kk]] = (int16_t)extend(br.bits(sz), sz);
            } else if (run == 15) {
              kk += 15;
            } else {
              break;
            }
          }
        }
    }
    if (++mx == J.mcus_x) { mx = 0; ++my; }
  }
  if (bad) { A.status[s].value = k; A.status[s].kind = JST_BAD_CODE; }
}

// ------------------------------------------------------------------- J3
// Thread per 8x8 block: dequantize + islow IDCT (13-bit constants, 2 pass-1
// bits) entirely in registers, 8 x 8-byte row stores into the component plane.
constexpr int kIdctThreads = 128;

__device__ __forceinline__ uint32_t range_out(int v) {   // post-IDCT range_limit[v & 1023]
  int s = ((v & 1023) ^ 512) - 512 + 128;
  return (uint32_t)min(max(s, 0), 255);
}

template <bool kPass1>
__device__ __forceinline__ void idct_1d(int& x0, int& x1, int& x2, int& x3, int& x4, int& x5, int& x6, int& x7) {
  // one column (pass 1) or row (pass 2); outputs descaled, pass 2 not yet range-limited
  constexpr int CB = 13, P1 = 2, SH = kPass1 ? CB - P1 : CB + P1 + 3;
  constexpr long long RND = 1ll << (SH - 1);
  long long z1, z2, z3, z4, z5, t0, t1, t2, t3, t10, t11, t12, t13;
  z2 = x2; z3 = x6;
  z1 = (z2 + z3) * 4433;
  t2 = z1 + z3 * -15137;
  t3 = z1 + z2 * 6270;
  t0 = ((long long)x0 + x4) * (1 << CB);
  t1 = ((long long)x0 - x4) * (1 << CB);
  t10 = t0 + t3; t13 = t0 - t3; t11 = t1 + t2; t12 = t1 - t2;
  t0 = x7; t1 = x5; t2 = x3; t3 = x1;
  z1 = t0 + t3; z2 = t1 + t2; z3 = t0 + t2; z4 = t1 + t3;
  z5 = (z3 + z4) * 9633;
  t0 *= 2446; t1 *= 16819; t2 *= 25172; t3 *= 12299;
  z1 *= -7373; z2 *= -20995; z3 *= -16069; z4 *= -3196;
  z3 += z5; z4 += z5;
  t0 += z1 + z3; t1 += z2 + z4; t2 += z2 + z3; t3 += z1 + z4;
  x0 = (int)((t10 + t3 + RND) >> SH); x7 = (int)((t10 - t3 + RND) >> SH);
  x1 = (int)((t11 + t2 + RND) >> SH); x6 = (int)((t11 - t2 + RND) >> SH);
  x2 = (int)((t12 + t1 + RND) >> SH); x5 = (int)((t12 - t1 + RND) >> SH);
  x3 = (int)((t13 + t0 + RND) >> SH); x4 = (int)((t13 - t0 + RND) >> SH);
}

__global__ void __launch_bounds__(kIdctThreads) jpeg_idct_kernel(const JpegArgs A) {
  const uint64_t b = (uint64_t)blockIdx.x * kIdctThreads + threadIdx.x;
  if (b >= A.total_blocks) return;
  const int s = find_sample(A.blk_prefix, A.count, b);
  const JpegDesc& J = A.jd[s];
  const uint32_t rel = (uint32_t)(b - J.blk_base);
  int c = 0;
  if (J.ncomp > 1 && rel >= J.comp[1].blk_off) c = (J.ncomp > 2 && rel >= J.comp[2].blk_off) ? 2 : 1;
  const JComp& C = J.comp[c];
  const uint32_t cb = rel - C.blk_off, by = cb / C.bw, bx = cb - by * C.bw;
  const uint4* src = reinterpret_cast<const uint4*>(A.coef + b * 64);
  const uint4* q4 = reinterpret_cast<const uint4*>(A.quant[C.q].q);
  int w[64];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint4 cv = __ldg(src + r), qv = __ldg(q4 + r);
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w}, qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[r * 8 + 2 * j] = (int)(int16_t)(cw[j] & 0xFFFF) * (int)(qw[j] & 0xFFFF);
      w[r * 8 + 2 * j + 1] = (int)(int16_t)(cw[j] >> 16) * (int)(qw[j] >> 16);
    }
  }
#pragma unroll
  for (int col = 0; col < 8; ++col) {
    int* x = w + col;
    if ((x[8] | x[16] | x[24] | x[32] | x[40] | x[48] | x[56]) == 0) {
      const int dc = x[0] * 4;
#pragma unroll
      for (int r = 0; r < 8; ++r) x[r * 8] = dc;
    } else {
      idct_1d<true>(x[0], x[8], x[16], x[24], x[32], x[40], x[48], x[56]);
    }
  }
  uint8_t* plane = A.planes + (J.blk_base + C.blk_off) * 64;
  const uint32_t pw = (uint32_t)C.bw * 8;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int* x = w + r * 8;
    uint32_t o[8];
    if ((x[1] | x[2] | x[3] | x[4] | x[5] | x[6] | x[7]) == 0) {
      const uint32_t v = range_out((x[0] + 16) >> 5);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = v;
    } else {
      idct_1d<false>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = range_out(x[j]);
    }
    const uint2 pk = make_uint2(o[0] | o[1] << 8 | o[2] << 16 | o[3] << 24, o[4] | o[5] << 8 | o[6] << 16 | o[7] << 24);
    *reinterpret_cast<uint2*>(plane + (size_t)(by * 8 + r) * pw + bx * 8) = pk;
  }
}

// ------------------------------------------------------------------- J4
// Thread per output pixel: libjpeg's fancy upsampling (h2v1 / h1v2 / h2v2
// triangle filters with edge replication; box when the downsampled width is
// <= 2) and JFIF YCbCr -> RGB in 16-bit fixed point.
constexpr int kColorThreads = 256;

__device__ __forceinline__ int comp_sample(const uint8_t* P, const JComp& c, int hmax, int vmax, int y, int x) {
  const int pw = c.bw * 8;
  const int rh = hmax / c.h, rv = vmax / c.v;
  auto at = [&](int yy, int xx) { return (int)__ldg(P + (size_t)yy * pw + xx); };
  if (rh == 1 && rv == 1) return at(y, x);
  const bool fancy_w = c.dw > 2;
  if (rv == 1) {                                    // h2v1
    const int j = x >> 1;
    if (!fancy_w) return at(y, j);
    if (x & 1) return (3 * at(y, j) + at(y, min(j + 1, (int)c.dw - 1)) + 2) >> 2;
    return (3 * at(y, j) + at(y, max(j - 1, 0)) + 1) >> 2;
  }
  const int i = y >> 1;
  const int i1 = (y & 1) ? min(i + 1, (int)c.dh - 1) : max(i - 1, 0);
  if (rh == 1) return (3 * at(i, x) + at(i1, x) + ((y & 1) ? 2 : 1)) >> 2;   // h1v2
  const int j = x >> 1;                             // h2v2
  if (!fancy_w) return at(i, j);
  const int jn = (x & 1) ? min(j + 1, (int)c.dw - 1) : max(j - 1, 0);
  const int cs = 3 * at(i, j) + at(i1, j), ns = 3 * at(i, jn) + at(i1, jn);
  return (3 * cs + ns + ((x & 1) ? 7 : 8)) >> 4;
}

__global__ void __launch_bounds__(kColorThreads) jpeg_color_kernel(const JpegArgs A) {
  const int s = blockIdx.y;
  const JpegDesc& J = A.jd[s];
  if (J.n_int == 0) return;
  const SampleDesc* d = sdesc(A, s);
  const int w = d->w, h = d->h;
  const int pix = blockIdx.x * kColorThreads + threadIdx.x;
  if (pix >= w * h) return;
  const int y = pix / w, x = pix - y * w;
  const uint8_t* planes = A.planes + J.blk_base * 64;
  uint8_t* out = A.scratch + (size_t)s * A.scratch_bytes;
  const int hmax = J.hmax, vmax = J.vmax;
  const int Y = comp_sample(planes + (size_t)J.comp[0].blk_off * 64, J.comp[0], hmax, vmax, y, x);
  if (J.ncomp == 1) { out[pix] = (uint8_t)Y; return; }
  const int cb = comp_sample(planes + (size_t)J.comp[1].blk_off * 64, J.comp[1], hmax, vmax, y, x) - 128;
  const int cr = comp_sample(planes + (size_t)J.comp[2].blk_off * 64, J.comp[2], hmax, vmax, y, x) - 128;
  const int r = Y + ((91881 * cr + 32768) >> 16);
  const int g = Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16);
  const int bl = Y + ((116130 * cb + 32768) >> 16);
  uint8_t* o = out + (size_t)pix * 3;
  o[0] = (uint8_t)min(max(r, 0), 255);
  o[1] = (uint8_t)min(max(g, 0), 255);
  o[2] = (uint8_t)min(max(bl, 0), 255);
}

int launch_jpeg(const JpegArgs& A, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (A.count <= 0 || A.total_int == 0) return 0;
  jpeg_scan_kernel<<<(A.count + kScanWarps - 1) / kScanWarps, 32 * kScanWarps, 0, st>>>(A);
  jpeg_huffman_kernel<<<(A.total_int + kHuffThreads - 1) / kHuffThreads, kHuffThreads, 0, st>>>(A);
  jpeg_idct_kernel<<<(unsigned)((A.total_blocks + kIdctThreads - 1) / kIdctThreads), kIdctThreads, 0, st>>>(A);
  dim3 g((A.max_pixels + kColorThreads - 1) / kColorThreads, A.count);
  jpeg_color_kernel<<<g, kColorThreads, 0, st>>>(A);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace bbx
