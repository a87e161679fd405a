// sm_100a JPEG decoder (codec id 3) — the decode stage of Decode /
// RandomResizedCrop / CenterCrop on JPEG samples.  See jpeg.h for the
// pipeline (J1 unstuff, J2 Huffman, J3 IDCT + upsample + color) and
// DESIGN.md §4 for what bounds each step.
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
__device__ __forceinline__ uint32_t align4(uint32_t x) { return (x + 3u) & ~3u; }
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------------- J1
// Warp per sample, 512 bytes of the entropy-coded segment per round (16 per
// lane).  Byte j is coded data unless it follows 0xFF (stuffing 0x00 or a
// marker code) or is an 0xFF that starts a marker; (0xFF, 0xD0..D7) is a
// restart marker and opens the next interval at the next 4-byte boundary of
// the output; any other marker ends the scan data.  A lane's effect on the
// output cursor is x -> x + a, or x -> align4(x + a) + c once it holds a
// marker; that family is closed under composition, so one warp scan gives
// every lane its starting cursor.
constexpr int kUnstuffWarps = 4;

struct CursorFn { uint32_t aligned, a, c; };   // aligned ? align4(x + a) + c : x + a

__device__ __forceinline__ CursorFn compose(CursorFn f, CursorFn g) {   // g after f
  if (!g.aligned) return f.aligned ? CursorFn{1u, f.a, f.c + g.a} : CursorFn{0u, f.a + g.a, 0u};
  return f.aligned ? CursorFn{1u, f.a, align4(f.c + g.a) + g.c} : CursorFn{1u, f.a + g.a, g.c};
}
__device__ __forceinline__ uint32_t apply(CursorFn f, uint32_t x) { return f.aligned ? align4(x + f.a) + f.c : x + f.a; }

__global__ void __launch_bounds__(32 * kUnstuffWarps) jpeg_unstuff_kernel(const JpegArgs A) {
  const int s = blockIdx.x * kUnstuffWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (s >= A.count) return;
  const JpegDesc& J = A.jd[s];
  const uint32_t nint = J.n_int;
  if (nint == 0) return;
  const uint8_t* base = A.payload + sdesc(A, s)->src;
  uint8_t* out = A.bits + J.bs_base;
  uint32_t* st = A.istart + J.int_base;
  uint32_t* en = A.iend + J.int_base;
  if (lane == 0) st[0] = 0;
  const uintptr_t ab = reinterpret_cast<uintptr_t>(base);
  const uintptr_t a_lo = ab + J.scan_off, a_hi = ab + J.scan_end;
  uint32_t kcur = 0, xcur = 0, carry = 0;
  bool seq_bad = false, done = false;
  uintptr_t c = a_lo & ~uintptr_t(15);
  uint4 vn = make_uint4(0, 0, 0, 0);                 // next round's chunk, loaded one round ahead
  if (c + (uintptr_t)lane * 16 < a_hi) vn = ld_nc_v4(reinterpret_cast<const void*>(c + (uintptr_t)lane * 16));
  for (; c < a_hi && !done; c += 512) {
    const uintptr_t my = c + (uintptr_t)lane * 16;
    const uint4 v = vn;
    vn = make_uint4(0, 0, 0, 0);
    if (my + 512 < a_hi) vn = ld_nc_v4(reinterpret_cast<const void*>(my + 512));   // >= 16 B tail padding
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t prev = __shfl_up_sync(0xffffffffu, w[3] >> 24, 1);
    if (lane == 0) prev = carry;
    uint32_t nxt = __shfl_down_sync(0xffffffffu, w[0] & 0xFF, 1);
    const uint32_t nxt31 = __shfl_sync(0xffffffffu, vn.x & 0xFF, 0);   // first byte of the next round
    if (lane == 31) nxt = nxt31;
    uint32_t keep = 0, rst = 0, term = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uintptr_t pos = my + j;
      const uint32_t b = (w[j >> 2] >> ((j & 3) * 8)) & 0xFF;
      const uint32_t p = pos == a_lo ? 0u : (j ? (w[(j - 1) >> 2] >> (((j - 1) & 3) * 8)) & 0xFF : prev);
      uint32_t n = j < 15 ? (w[(j + 1) >> 2] >> (((j + 1) & 3) * 8)) & 0xFF : nxt;
      if (pos + 1 >= a_hi) n = 0xD9;
      if (pos < a_lo || pos >= a_hi) continue;
      const bool marker = b == 0xFF && n != 0x00;
      if (p != 0xFF && !marker) keep |= 1u << j;
      if (marker && (n & 0xF8) == 0xD0) rst |= 1u << j;
      if (marker && n != 0xFF && (n & 0xF8) != 0xD0) term |= 1u << j;
    }
    // everything from the first non-RST marker on is not scan data
    const uint32_t tb = __ballot_sync(0xffffffffu, term != 0);
    if (tb) {
      const int fl = __ffs(tb) - 1;
      if (lane > fl) { keep = 0; rst = 0; }
      if (lane == fl) { const uint32_t m = (1u << (__ffs(term) - 1)) - 1; keep &= m; rst &= m; }
      done = true;
    }
    // this lane's cursor function, then an inclusive warp scan of them
    CursorFn f{0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (rst >> j & 1) f = f.aligned ? CursorFn{1u, f.a, align4(f.c)} : CursorFn{1u, f.a, 0u};
      if (keep >> j & 1) { if (f.aligned) ++f.c; else ++f.a; }
    }
    uint32_t nr = __popc(rst), nr_incl = nr;
    CursorFn inc = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      CursorFn e{__shfl_up_sync(0xffffffffu, inc.aligned, o), __shfl_up_sync(0xffffffffu, inc.a, o),
                 __shfl_up_sync(0xffffffffu, inc.c, o)};
      const uint32_t r = __shfl_up_sync(0xffffffffu, nr_incl, o);
      if (lane >= o) { inc = compose(e, inc); nr_incl += r; }
    }
    CursorFn exc{__shfl_up_sync(0xffffffffu, inc.aligned, 1), __shfl_up_sync(0xffffffffu, inc.a, 1),
                 __shfl_up_sync(0xffffffffu, inc.c, 1)};
    if (lane == 0) exc = CursorFn{0u, 0u, 0u};
    uint32_t x = apply(exc, xcur), k = kcur + nr_incl - nr;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (rst >> j & 1) {
        const uint32_t n = (j < 15 ? (w[(j + 1) >> 2] >> (((j + 1) & 3) * 8)) : nxt) & 7;
        if (n != (k & 7)) seq_bad = true;
        if (k + 1 < nint) { en[k] = x; st[k + 1] = align4(x); }
        x = align4(x);
        ++k;
      }
      if (keep >> j & 1) out[x++] = (uint8_t)(w[j >> 2] >> ((j & 3) * 8));
    }
    const CursorFn all{__shfl_sync(0xffffffffu, inc.aligned, 31), __shfl_sync(0xffffffffu, inc.a, 31),
                       __shfl_sync(0xffffffffu, inc.c, 31)};
    xcur = apply(all, xcur);
    kcur += __shfl_sync(0xffffffffu, nr_incl, 31);
    carry = __shfl_sync(0xffffffffu, w[3] >> 24, 31);
  }
  seq_bad = __any_sync(0xffffffffu, seq_bad);
  if (lane == 0) {
    SampleStatus& S = A.status[s];
    S.kind = 0; S.value = 0;
    if (kcur != nint - 1) { S.kind = JST_MARKER_COUNT; S.value = kcur; }
    else if (seq_bad) S.kind = JST_MARKER_SEQ;
    else en[nint - 1] = xcur;
  }
}

// ------------------------------------------------------------------- J2
// Thread per restart interval (DC predictors restart at zero, T.81
// F.2.1.3.1), one symbol per loop iteration whatever block / MCU it belongs
// to.  The body is branch-free except at block ends and for codes longer than
// the fast table, so the lanes of a warp stay converged: the 32-bit refill is
// predicated, the extra bits are always extracted (0 of them for EOB / ZRL),
// and only nonzero coefficients are stored into the pre-zeroed block.  Past
// the interval's end the stream reads as zeros (libjpeg's rule once a marker
// is reached).
constexpr int kHuffThreads = 128;

template <typename T>
__device__ __forceinline__ int find_sample(const T* prefix, int count, T t) {   // largest s: prefix[s] <= t
  int lo = 0, hi = count;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(&prefix[mid]) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename T>
__device__ __forceinline__ T sel3(int i, T a, T b, T c) { return i == 0 ? a : (i == 1 ? b : c); }

__global__ void __launch_bounds__(kHuffThreads) jpeg_huffman_kernel(const JpegArgs A) {
  extern __shared__ __align__(16) uint32_t sfast[];
  __shared__ uint8_t nat[80];
  constexpr int TW = 1 << kJpegFastBits;
  const bool smem_tabs = A.n_huff <= kJpegSmemTables;
  if (smem_tabs) {
    const int n = A.n_huff * TW;
    for (int i = threadIdx.x; i < n; i += kHuffThreads) sfast[i] = __ldg(&A.huff[i / TW].fast[i % TW]);
  }
  for (int i = threadIdx.x; i < 80; i += kHuffThreads) nat[i] = c_natural[i];
  __syncthreads();
  const uint32_t t = blockIdx.x * kHuffThreads + threadIdx.x;
  if (t >= A.total_int) return;
  const int s = find_sample(A.int_prefix, A.count, t);
  if (A.status[s].kind != 0) return;                 // J1 rejected the marker layout
  const JpegDesc& J = A.jd[s];
  const uint32_t k = t - J.int_base;
  const uint32_t mcus_x = J.mcus_x, total = mcus_x * J.mcus_y;
  const uint32_t m0 = k * J.restart, m1 = min(m0 + J.restart, total);
  if (m0 >= m1) return;
  const uint64_t sched = J.sched;
  const int bpm = J.bpm;
  // per-component constants (selected by index: no local-memory arrays)
  const uint32_t bw0 = J.comp[0].bw, bw1 = J.comp[1].bw, bw2 = J.comp[2].bw;
  const uint32_t of0 = J.comp[0].blk_off, of1 = J.comp[1].blk_off, of2 = J.comp[2].blk_off;
  const uint32_t hv0 = J.comp[0].h | J.comp[0].v << 8, hv1 = J.comp[1].h | J.comp[1].v << 8,
                 hv2 = J.comp[2].h | J.comp[2].v << 8;
  const uint32_t tb0 = J.comp[0].dc | (uint32_t)J.comp[0].ac << 16, tb1 = J.comp[1].dc | (uint32_t)J.comp[1].ac << 16,
                 tb2 = J.comp[2].dc | (uint32_t)J.comp[2].ac << 16;
  int16_t* const coef = A.coef + J.blk_base * 64;

  const uint32_t* wp = reinterpret_cast<const uint32_t*>(A.bits + J.bs_base + A.istart[t]);
  int rem = (int)(A.iend[t] - A.istart[t]);
  uint64_t acc = 0;
  int nb = 0;

  uint32_t m = m0, mx = m0 % mcus_x, my = m0 / mcus_x;
  int b = 0, kk = 0, ci = 0;
  int pred0 = 0, pred1 = 0, pred2 = 0;
  const uint32_t* fdc = nullptr;
  const uint32_t* fac = nullptr;
  const JHuff* gdc = nullptr;
  const JHuff* gac = nullptr;
  int16_t* cb = nullptr;
  bool bad = false;
  auto setup = [&]() {                               // block b of MCU (mx, my)
    const uint32_t e = (uint32_t)(sched >> (4 * b)) & 15u;
    ci = (int)(e & 3);
    const uint32_t hv = sel3(ci, hv0, hv1, hv2), H = hv & 0xFF, V = hv >> 8;
    const uint32_t bidx =
        sel3(ci, of0, of1, of2) + (my * V + ((e >> 2) & 1)) * sel3(ci, bw0, bw1, bw2) + mx * H + (e >> 3);
    cb = coef + (size_t)bidx * 64;
    const uint32_t tb = sel3(ci, tb0, tb1, tb2);
    gdc = A.huff + (tb & 0xFFFF);
    gac = A.huff + (tb >> 16);
    fdc = smem_tabs ? sfast + (tb & 0xFFFF) * TW : gdc->fast;
    fac = smem_tabs ? sfast + (tb >> 16) * TW : gac->fast;
    kk = 0;
  };
  setup();
  for (;;) {
    {                                                // predicated 32-bit refill
      const bool need = nb <= 32;
      uint32_t wv = __byte_perm(__ldg(wp), 0, 0x0123);
      const uint32_t keep = rem >= 4 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : (0xFFFFFFFFu << (8 * (4 - rem))));
      wv = need ? (wv & keep) : 0u;
      acc |= (uint64_t)wv << (need ? 32 - nb : 0);
      wp += (need && rem > 4) ? 1 : 0;
      rem -= need ? 4 : 0;
      nb += need ? 32 : 0;
    }
    const uint32_t e = (kk ? fac : fdc)[(uint32_t)(acc >> (64 - kJpegFastBits))];
    int len, size, run;
    bool eob;
    if (e & kFastValid) {
      len = (int)(e & 31);
      size = (int)((e >> 5) & 31);
      run = (int)((e >> 10) & 15);
      eob = (e & kFastEob) != 0;
    } else {                                         // code longer than the fast table
      const JHuff* g = kk ? gac : gdc;
      const uint32_t c16 = (uint32_t)(acc >> 48);
      len = kJpegFastBits + 1;
      while (len <= 16 && (int32_t)(c16 >> (16 - len)) > __ldg(&g->maxcode[len])) ++len;
      if (len > 16) { bad = true; break; }
      const int sym = __ldg(&g->vals[(c16 >> (16 - len)) + __ldg(&g->valoff[len])]);
      size = kk ? (sym & 15) : sym;
      run = kk ? (sym >> 4) : 0;
      eob = kk && size == 0 && run != 15;
    }
    acc <<= len;
    nb -= len;
    const uint32_t bits = size ? (uint32_t)(acc >> (64 - size)) : 0u;
    acc <<= size;
    nb -= size;
    int v = (int)bits;
    if (size && bits < (1u << (size - 1))) v -= (1 << size) - 1;   // EXTEND (F.2.2.1)
    if (kk == 0) {                                   // DC: prediction per component
      v += sel3(ci, pred0, pred1, pred2);
      pred0 = ci == 0 ? v : pred0;
      pred1 = ci == 1 ? v : pred1;
      pred2 = ci == 2 ? v : pred2;
    }
    const int pos = kk + run;
    if (v != 0) cb[nat[pos]] = (int16_t)v;
    kk = eob ? 64 : pos + 1;
    if (kk >= 64) {                                  // block done: next block of the MCU / next MCU
      if (++b == bpm) {
        b = 0;
        ++m;
        if (++mx == mcus_x) { mx = 0; ++my; }
        if (m >= m1) break;
      }
      setup();
    }
  }
  if (bad) { A.status[s].value = k; A.status[s].kind = JST_BAD_CODE; }
}

// ------------------------------------------------------------------- J3
// CTA per (sample, MCU row).  Phase 1: one thread per 8x8 block, dequantize +
// islow IDCT (13-bit constants, 2 pass-1 bits) in registers, rows into the
// component's shared-memory window.  Phase 2: one thread per output pixel:
// libjpeg's fancy upsampling (h2v1 / h1v2 / h2v2 triangle filters with edge
// replication; box when the downsampled width is <= 2) and JFIF YCbCr -> RGB
// in 16-bit fixed point, into the decode scratch (HWC, row stride w*C).
constexpr int kPixThreads = 256;

__device__ __forceinline__ uint32_t range_out(int v) {   // post-IDCT range_limit[v & 1023]
  int s = ((v & 1023) ^ 512) - 512 + 128;
  return (uint32_t)min(max(s, 0), 255);
}

template <bool kPass1>
__device__ __forceinline__ void idct_1d(int& x0, int& x1, int& x2, int& x3, int& x4, int& x5, int& x6, int& x7) {
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

// One block: coefficients (global, natural order) -> 8 rows of 8 bytes at dst (stride bytes).
__device__ __forceinline__ void idct_block(const int16_t* coef, const uint16_t* q, uint8_t* dst, int stride) {
  const uint4* src = reinterpret_cast<const uint4*>(coef);
  const uint4* q4 = reinterpret_cast<const uint4*>(q);
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
    *reinterpret_cast<uint2*>(dst + (size_t)r * stride) =
        make_uint2(o[0] | o[1] << 8 | o[2] << 16 | o[3] << 24, o[4] | o[5] << 8 | o[6] << 16 | o[7] << 24);
  }
}

struct Win {                       // one component's shared-memory window for an MCU row
  const uint8_t* p;
  int y0, pw, dw, dh, rh, rv;      // plane row of window row 0, row pitch, downsampled dims, up ratios
};

__device__ __forceinline__ int win_sample(const Win& c, int y, int x) {
  auto at = [&](int yy, int xx) { return (int)c.p[(yy - c.y0) * c.pw + xx]; };
  if (c.rh == 1 && c.rv == 1) return at(y, x);
  const bool fancy_w = c.dw > 2;
  if (c.rv == 1) {                                  // h2v1
    const int j = x >> 1;
    if (!fancy_w) return at(y, j);
    if (x & 1) return (3 * at(y, j) + at(y, min(j + 1, c.dw - 1)) + 2) >> 2;
    return (3 * at(y, j) + at(y, max(j - 1, 0)) + 1) >> 2;
  }
  const int i = y >> 1;
  const int i1 = (y & 1) ? min(i + 1, c.dh - 1) : max(i - 1, 0);
  if (c.rh == 1) return (3 * at(i, x) + at(i1, x) + ((y & 1) ? 2 : 1)) >> 2;   // h1v2
  const int j = x >> 1;                             // h2v2
  if (!fancy_w) return at(i, j);
  const int jn = (x & 1) ? min(j + 1, c.dw - 1) : max(j - 1, 0);
  const int cs = 3 * at(i, j) + at(i1, j), ns = 3 * at(i, jn) + at(i1, jn);
  return (3 * cs + ns + ((x & 1) ? 7 : 8)) >> 4;
}

__global__ void __launch_bounds__(kPixThreads) jpeg_pixels_kernel(const JpegArgs A) {
  extern __shared__ __align__(16) uint8_t psm[];
  const int s = blockIdx.y, r = blockIdx.x;
  const JpegDesc& J = A.jd[s];
  if (J.n_int == 0 || r >= J.mcus_y || A.status[s].kind != 0) return;
  const SampleDesc* d = sdesc(A, s);
  const int w = d->w, h = d->h, nc = J.ncomp, hmax = J.hmax, vmax = J.vmax;
  Win win[3];
  int brlo[3], brhi[3], njob[3];
  int off = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (c >= nc) { njob[c] = 0; continue; }
    const JComp& C = J.comp[c];
    const int rv = vmax / C.v, ext = rv == 2 ? 1 : 0;
    win[c].p = psm + off;
    win[c].y0 = (r * C.v - ext) * 8;
    win[c].pw = C.bw * 8;
    win[c].dw = C.dw; win[c].dh = C.dh; win[c].rh = hmax / C.h; win[c].rv = rv;
    brlo[c] = max(r * C.v - ext, 0);
    brhi[c] = min(r * C.v + C.v - 1 + ext, (int)C.bh - 1);
    njob[c] = (brhi[c] - brlo[c] + 1) * C.bw;
    off += jpeg_window_rows(C.v, vmax) * C.bw * 8;
  }
  const int16_t* coef = A.coef + J.blk_base * 64;
  for (int jb = threadIdx.x; jb < njob[0] + njob[1] + njob[2]; jb += kPixThreads) {
    int c = 0, q = jb;
    if (q >= njob[0]) { q -= njob[0]; c = 1; if (q >= njob[1]) { q -= njob[1]; c = 2; } }
    const JComp& C = J.comp[c];
    const int br = brlo[c] + q / C.bw, bx = q - (q / C.bw) * C.bw;
    idct_block(coef + ((size_t)C.blk_off + (size_t)br * C.bw + bx) * 64, A.quant[C.q].q,
               psm + (win[c].p - psm) + (br * 8 - win[c].y0) * win[c].pw + bx * 8, win[c].pw);
  }
  __syncthreads();
  const int y_first = r * vmax * 8, rows = min(vmax * 8, h - y_first);
  uint8_t* outp = A.scratch + (size_t)s * A.scratch_bytes;
  if (nc == 3 && hmax == 2 && vmax == 2 && win[0].rh == 1 && win[0].rv == 1 && win[1].rh == 2 &&
      win[1].rv == 2 && win[2].rh == 2 && win[2].rv == 2 && win[1].dw > 2 && win[2].dw > 2) {
    // 4:2:0 (h2v2 fancy): a thread produces the two output pixels of one chroma column
    const int cw = (w + 1) >> 1, dw = win[1].dw, dh = win[1].dh, cpw = win[1].pw;
    for (int idx = threadIdx.x; idx < rows * cw; idx += kPixThreads) {
      const int yy = idx / cw, j = idx - yy * cw, y = y_first + yy;
      const int i = y >> 1, i1 = (y & 1) ? min(i + 1, dh - 1) : max(i - 1, 0);
      const int jl = max(j - 1, 0), jr = min(j + 1, dw - 1);
      const int ra = (i - win[1].y0) * cpw, rb = (i1 - win[1].y0) * cpw;
      int ce[2], co[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint8_t* P = win[1 + q].p;
        const int cs = 3 * P[ra + j] + P[rb + j], cl = 3 * P[ra + jl] + P[rb + jl], cr = 3 * P[ra + jr] + P[rb + jr];
        ce[q] = ((3 * cs + cl + 8) >> 4) - 128;
        co[q] = ((3 * cs + cr + 7) >> 4) - 128;
      }
      const uint8_t* yrow = win[0].p + (y - win[0].y0) * win[0].pw;
      uint8_t* o = outp + ((size_t)y * w + 2 * j) * 3;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (2 * j + q >= w) break;
        const int Y = yrow[2 * j + q], cb = q ? co[0] : ce[0], cr = q ? co[1] : ce[1];
        o[3 * q] = (uint8_t)min(max(Y + ((91881 * cr + 32768) >> 16), 0), 255);
        o[3 * q + 1] = (uint8_t)min(max(Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16), 0), 255);
        o[3 * q + 2] = (uint8_t)min(max(Y + ((116130 * cb + 32768) >> 16), 0), 255);
      }
    }
    return;
  }
  for (int idx = threadIdx.x; idx < rows * w; idx += kPixThreads) {
    const int yy = idx / w, x = idx - yy * w, y = y_first + yy;
    const int Y = win_sample(win[0], y, x);
    if (nc == 1) { outp[(size_t)y * w + x] = (uint8_t)Y; continue; }
    const int cb = win_sample(win[1], y, x) - 128, cr = win_sample(win[2], y, x) - 128;
    uint8_t* o = outp + ((size_t)y * w + x) * 3;
    o[0] = (uint8_t)min(max(Y + ((91881 * cr + 32768) >> 16), 0), 255);
    o[1] = (uint8_t)min(max(Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16), 0), 255);
    o[2] = (uint8_t)min(max(Y + ((116130 * cb + 32768) >> 16), 0), 255);
  }
}

int launch_jpeg(const JpegArgs& A, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (A.count <= 0 || A.total_int == 0) return 0;
  jpeg_unstuff_kernel<<<(A.count + kUnstuffWarps - 1) / kUnstuffWarps, 32 * kUnstuffWarps, 0, st>>>(A);
  const int hsmem = A.n_huff <= kJpegSmemTables ? A.n_huff * (int)sizeof(JHuff::fast) : 0;
  if (hsmem > 48 * 1024) cudaFuncSetAttribute(jpeg_huffman_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem);
  jpeg_huffman_kernel<<<(A.total_int + kHuffThreads - 1) / kHuffThreads, kHuffThreads, hsmem, st>>>(A);
  if (A.pix_smem > 48 * 1024)
    cudaFuncSetAttribute(jpeg_pixels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, A.pix_smem);
  jpeg_pixels_kernel<<<dim3(A.max_mcu_rows, A.count), kPixThreads, A.pix_smem, st>>>(A);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace bbx
