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

// ------------------------------------------------------------------- J2
// Thread per restart interval (DC predictors restart at zero, T.81
// F.2.1.3.1), one symbol per loop iteration whatever block / MCU it belongs
// to, so the lanes of a warp stay converged.  Per iteration: a predicated
// 32-bit refill from two 16-byte chunks held in registers (the next one is
// loaded a chunk ahead; J1 left zero padding after every interval, so reading
// past the data yields zeros, libjpeg's rule once a marker is reached), one u16 table
// lookup for code length / extra bits / run / EOB, extra-bit extraction with
// a branch-free EXTEND, and a store of the coefficient when it is nonzero
// (the block buffer is pre-zeroed).  Block ends read the next block's
// component / offset / tables from a per-thread slot table in shared memory.
constexpr int kHuffThreads = 256;           // 8 warps share one copy of the smem tables
constexpr int kHuffCtasPerSm = 3;           // a batch of 1024 ImageNet-sized JPEGs has ~110k intervals: ~3 CTAs
                                            // per SM hold all of them at once (4 / 5 measured the same)
constexpr int kExtraSymbols = 4;   // AC symbols decoded after the first in one iteration
                                   // (A/B, configs[2] value: 2 / 4 / 6 / 8 -> 2.65 / 2.73 / 2.65 / 2.51 M img/s;
                                   // branch-free extras: 3 / 4 / 5 / 6 -> J2 324 / 313 / 316 / 334 us under ncu)
// Each lane assembles its current 8x8 block in shared memory and writes it to the
// coefficient buffer with one 128-byte bulk copy (cp.async.bulk, async proxy) when
// the block ends: scattered 2-byte global stores of single coefficients kept the L1
// busy with one sector per lane per coefficient, and the buffer needed a memset
// first; eight 16-byte stores per block through the L1 cost the two-stream pipeline
// 10 % against the bulk copy (configs[2] device time 0.634 -> 0.571 ms per batch).
// 144-byte lane stride: the lanes' 2-byte coefficient stores spread over the banks.
constexpr int kBlkStride = 144;
__host__ __device__ constexpr int huff_blk_bytes() { return kHuffThreads * kBlkStride; }
constexpr int kMaxBpm = 12;                 // blocks per MCU with sampling factors <= 2


template <typename T>
__device__ __forceinline__ T sel3(int i, T a, T b, T c) { return i == 0 ? a : (i == 1 ? b : c); }

template <bool kSmem>
__global__ void __launch_bounds__(kHuffThreads, kHuffCtasPerSm) jpeg_huffman_kernel(const JpegArgs A) {
  extern __shared__ __align__(16) uint8_t hsm[];
  constexpr int TW = 1 << kJpegFastBits;
  constexpr uint32_t TSTRIDE = kSmem ? TW : (uint32_t)(sizeof(JHuff) / 4);
  const int tabs_bytes = kSmem ? A.n_huff * TW * 4 : 0;
  const uint32_t* tab = kSmem ? reinterpret_cast<const uint32_t*>(hsm + huff_blk_bytes())
                              : reinterpret_cast<const uint32_t*>(A.huff);
  // long codes (12..16 bits): per table maxcode[12..16], valoff[12..16] (int32) and vals[256] in smem
  constexpr int kSlowBytes = 10 * 4 + 256;
  uint8_t* slow = hsm + huff_blk_bytes() + tabs_bytes;
  int16_t* myblk = reinterpret_cast<int16_t*>(hsm + threadIdx.x * kBlkStride);   // this lane's block
  {
    uint4* z = reinterpret_cast<uint4*>(myblk);
#pragma unroll
    for (int j = 0; j < 8; ++j) z[j] = make_uint4(0, 0, 0, 0);
  }
  if (kSmem) {
    uint32_t* st = reinterpret_cast<uint32_t*>(hsm + huff_blk_bytes());
    const int n = A.n_huff * TW;
    for (int i = threadIdx.x; i < n; i += kHuffThreads) st[i] = __ldg(&A.huff[i / TW].fast[i % TW]);
    for (int i = threadIdx.x; i < A.n_huff * kSlowBytes; i += kHuffThreads) {
      const int tb = i / kSlowBytes, o = i % kSlowBytes;
      const JHuff& H = A.huff[tb];
      uint8_t v;
      if (o < 20) { const int32_t m = H.maxcode[12 + o / 4]; v = (uint8_t)(m >> (8 * (o & 3))); }
      else if (o < 40) { const int32_t m = H.valoff[12 + (o - 20) / 4]; v = (uint8_t)(m >> (8 * (o & 3))); }
      else v = H.vals[o - 40];
      slow[i] = v;
    }
  }
  // This CTA's intervals [c0, c0 + kHuffThreads) (A/B: taking every gridDim.x-th
  // interval instead balances the CTAs -- J2 alone 295 -> 280 us -- but lowers the
  // batch rate of the two-stream pipeline, 2.29 -> 2.24 M img/s, whose
  // overlapping batches fill the SMs a contiguous J2 leaves idle at its end),
  // ordered longest first so that each warp decodes intervals of similar length
  // (a warp runs until its longest lane finishes; interval lengths vary ~4x
  // within an image).  Key: stream bytes + 1 (0: outside the
  // region of interest or a rejected sample: never decoded) | position.
  __shared__ uint32_t skey[kHuffThreads], ssamp[kHuffThreads];
  const uint32_t c0 = blockIdx.x * kHuffThreads;
  {
    const uint32_t t = c0 + threadIdx.x;
    uint32_t key = 0, si = 0;
    if (t < A.total_int) {
      uint32_t lo = 0, hi = (uint32_t)A.count;       // the sample: int_prefix[si] <= t < int_prefix[si + 1]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&A.int_prefix[mid]) <= t) lo = mid; else hi = mid;
      }
      si = lo;
      const JpegDesc& J = A.jd[si];
      const uint32_t k = t - J.int_base;
      if (k < J.n_int && jpeg_interval_live(J, jpeg_mcu_rect(J), k)) {
        const uint32_t e = k + 1 < J.n_int ? __ldg(&A.starts[t + 1]) : J.scan_end;
        key = min(e - __ldg(&A.starts[t]) + 1u, 0xFFFFFFu) << 8;
      }
    }
    skey[threadIdx.x] = key | threadIdx.x;
    ssamp[threadIdx.x] = si;
  }
  __syncthreads();
#pragma unroll 1
  for (int kb = 2; kb <= kHuffThreads; kb <<= 1)      // bitonic sort, descending
#pragma unroll 1
    for (int j = kb >> 1; j > 0; j >>= 1) {
      const int ixj = threadIdx.x ^ j;
      if (ixj > (int)threadIdx.x) {
        const uint32_t a = skey[threadIdx.x], b = skey[ixj];
        if (((threadIdx.x & kb) == 0) ? a < b : a > b) { skey[threadIdx.x] = b; skey[ixj] = a; }
      }
      __syncthreads();
    }
  const uint32_t mine = skey[threadIdx.x];

  // per-lane decoder state of the current restart interval.  The reader
  // walks the stuffed entropy-coded bytes (T.81 F.1.2.3): a logical 32-bit
  // word = 4 stream bytes at the interval's byte phase (one PRMT of two
  // aligned words); words without 0xFF go straight into the bit buffer, any
  // other word byte by byte -- 0xFF 0x00 is a data 0xFF, 0xFF + anything else
  // is a marker (the next RSTn, EOI, or corruption) after which zeros are
  // supplied (libjpeg's fill_bit_buffer rule; oracle/jpeg_oracle.c get_bit).
  const uint32_t* wp = nullptr;                      // next aligned stream word to load
  uintptr_t wend = 0;                                // end of the sample's scan data (exclusive)
  uint32_t qn = 0;                                   // the word loaded one refill ahead
  uint32_t qa = 0, qb = 0, sel = 0x0123;            // window of two aligned words, PRMT selector
  bool carry = false, marker = false;               // pending 0xFF / marker reached
  uint64_t acc = 0;
  int nb = 0;
  uint32_t m = 0, m1 = 0;                            // MCU counter / end
  int b = 0, bpm = 1, kk = 0, ci = 0, s = 0;
  uint32_t k = 0, sched = 0, tdc = 0, tac = 0;
  uint64_t tabs = 0;                                 // dc / ac table ids of the components, 9 bits each
  int pred0 = 0, pred1 = 0, pred2 = 0;
  int16_t* cb = nullptr;

  // one aligned stream word: a predicated L1-allocating load (no branch, so the
  // lanes of a warp never diverge on it); bytes past the scan data read as 0xFF
  // (a marker), and no byte past the word holding the last one is loaded
  auto ld_word = [&](const uint32_t* p) -> uint32_t {
    const intptr_t rem = (intptr_t)(wend - reinterpret_cast<uintptr_t>(p));
    uint32_t w = ~0u;
    if (rem > 0) w = __ldg(p);
    return rem >= 4 ? w : (w | (~0u << (8 * (int)max(rem, (intptr_t)0))));
  };
  auto next_word = [&]() -> uint32_t {               // the next window word; the one after is loaded now
    const uint32_t w = qn;
    qn = ld_word(wp);
    ++wp;
    // the stream two lines ahead goes into L1 when a word starts a 128-B line
    if ((reinterpret_cast<uintptr_t>(wp) & 127) == 0 && reinterpret_cast<uintptr_t>(wp + 64) < wend)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(wp + 64));
    return w;
  };
  auto comp_tables = [&]() {                         // ci, tdc, tac of block b
    ci = (int)((sched >> (2 * b)) & 3u);
    const uint32_t ids = (uint32_t)(tabs >> (18 * ci));
    tdc = (ids & 511u) * TSTRIDE;
    tac = ((ids >> 9) & 511u) * TSTRIDE;
  };
  // set up interval t of sample si; false when it has nothing to decode
  auto start = [&](uint32_t t, int si) -> bool {
    s = si;
    const JpegDesc& J = A.jd[s];
    k = t - J.int_base;
    const uint32_t total = (uint32_t)J.mcus_x * J.mcus_y;
    m = k * J.restart;
    m1 = min(m + J.restart, total);
    if (m >= m1) return false;
    bpm = J.bpm;
    sched = 0;
    for (int q = 0; q < bpm; ++q) sched |= ((uint32_t)(J.sched >> (4 * q)) & 3u) << (2 * q);
    tabs = 0;
    for (int c = 0; c < J.ncomp; ++c) tabs |= (uint64_t)(J.comp[c].dc | (uint32_t)J.comp[c].ac << 9) << (18 * c);
    cb = A.coef + (J.blk_base + (uint64_t)m * bpm) * 64;
    const uint8_t* base = A.payload + sdesc(A, s)->src;
    const uintptr_t a = reinterpret_cast<uintptr_t>(base + __ldg(&A.starts[t]));
    wend = reinterpret_cast<uintptr_t>(base + J.scan_end);
    wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    if (reinterpret_cast<uintptr_t>(wp + 32) < wend) asm volatile("prefetch.global.L1 [%0];" ::"l"(wp + 32));
    if (reinterpret_cast<uintptr_t>(wp + 64) < wend) asm volatile("prefetch.global.L1 [%0];" ::"l"(wp + 64));
    qn = ld_word(wp);
    ++wp;
    const uint32_t ph = (uint32_t)(a & 3);
    sel = (ph << 12) | ((ph + 1) << 8) | ((ph + 2) << 4) | (ph + 3);   // big-endian bytes ph..ph+3 of (qa, qb)
    qa = next_word();
    qb = next_word();
    carry = marker = false;
    acc = 0; nb = 0;
    b = 0; kk = 0;
    pred0 = pred1 = pred2 = 0;
    comp_tables();
    return true;
  };
  bool active = (mine >> 8) != 0 && start(c0 + (mine & 0xFFu), (int)ssamp[mine & 0xFFu]);
  while (__any_sync(0xffffffffu, active)) {
    if (!active) continue;
    while (nb <= 32) {                               // refill: >= 33 valid bits for the symbol(s) below
      const uint32_t wv = __byte_perm(qa, qb, sel);
      if (!(carry | marker) && __vcmpeq4(wv, 0xFFFFFFFFu) == 0) {
        acc |= (uint64_t)wv << (32 - nb);
        nb += 32;
      } else if (marker) {                           // past a marker: zeros (acc's low bits are zero)
        nb += 32;
      } else {                                       // a 0xFF in the word: byte by byte, branch-free
        uint32_t o = 0;
        int no = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t by = (wv >> (24 - 8 * j)) & 0xFFu;
          // after a 0xFF: 0x00 is a data 0xFF, anything else a marker (zeros from there on)
          const bool mk = marker | (carry & (by != 0));
          const bool emit = mk | carry | (by != 0xFFu);
          const uint32_t ob = mk ? 0u : (carry ? 0xFFu : by);
          carry = !mk && !carry && by == 0xFFu;
          marker = mk;
          o = emit ? (o << 8) | ob : o;
          no += emit ? 1 : 0;
        }
        if (no) acc |= (uint64_t)o << (64 - nb - 8 * no);
        nb += 8 * no;
      }
      qa = qb;
      qb = next_word();
    }
    uint32_t e = tab[(kk ? tac : tdc) + (uint32_t)(acc >> (64 - kJpegFastBits))];
    bool bad = false;
    if (!(e & kFastValid)) {                         // code longer than the fast table (12..16 bits)
      const uint32_t tid = (kk ? tac : tdc) / TSTRIDE;
      const uint32_t c16 = (uint32_t)(acc >> 48);
      uint32_t hit = 0;
      if (kSmem) {
        const int32_t* mc = reinterpret_cast<const int32_t*>(slow + tid * kSlowBytes);
#pragma unroll
        for (int l = 12; l <= 16; ++l) hit |= ((int32_t)(c16 >> (16 - l)) <= mc[l - 12] ? 1u : 0u) << (l - 12);
      } else {
        const JHuff* g = A.huff + tid;
#pragma unroll
        for (int l = 12; l <= 16; ++l) hit |= ((int32_t)(c16 >> (16 - l)) <= __ldg(&g->maxcode[l]) ? 1u : 0u) << (l - 12);
      }
      int sym = 0, len = 16;
      if (hit == 0) bad = true;
      else {
        len = 11 + __ffs(hit);
        const int code = (int)(c16 >> (16 - len));
        if (kSmem) {
          const uint8_t* sb = slow + tid * kSlowBytes;
          sym = sb[40 + code + reinterpret_cast<const int32_t*>(sb + 20)[len - 12]];
        } else {
          const JHuff* g = A.huff + tid;
          sym = __ldg(&g->vals[code + __ldg(&g->valoff[len])]);
        }
      }
      const int size = kk ? (sym & 15) : sym, run = kk ? (sym >> 4) : 0;
      const uint32_t adv = (kk && size == 0 && run != 15) ? 64u : (uint32_t)run + 1u;
      e = kFastValid | (uint32_t)len << 25 | adv << kFastAdvShift | (uint32_t)size;
    }
    // common tail: consume the code (or code + extra bits), then any extra bits still pending
    const int used = (int)((e >> 25) & 31);
    acc <<= used;
    const int size = (e & kFastFull) ? 0 : (int)(e & 15u);
    const uint32_t hi = (uint32_t)(acc >> 32);
    const uint32_t bits = __funnelshift_l(hi, 0u, size);               // top `size` bits (0 when size == 0)
    const int sgn = (int)hi >> 31;                                      // leading extra bit 1: positive
    int v = (e & kFastFull) ? (int)(int16_t)(e & 0xFFFF)
                            : (int)bits + ((int)((0xFFFFFFFFu << size) + 1u) & ~sgn);   // EXTEND (F.2.2.1)
    acc <<= size;
    nb -= used + size;
    const int adv = (int)((e >> kFastAdvShift) & kFastAdvMask);
    if (kk == 0) {                                   // DC: prediction per component
      int p = ci == 0 ? pred0 : pred1;
      p = ci == 2 ? pred2 : p;
      v += p;
      pred0 = ci == 0 ? v : pred0;
      pred1 = ci == 1 ? v : pred1;
      pred2 = ci == 2 ? v : pred2;
    }
    const int pos = kk + adv - 1;
    if (v != 0 && !bad) myblk[min(pos, 63)] = (int16_t)v;   // zig-zag order (J3 de-zigzags at compile time)
    kk += adv;                                       // an end of block advances past 63
    // more AC symbols in the same iteration while the block continues and the
    // bit buffer holds the symbol with its value: code + extra bits within the
    // 11-bit peek (entries that need more extra bits wait for the next iteration).
    // Branch-free: every lane looks its entry up and consumes nothing when it may
    // not (nested ifs diverged per symbol: J2 354 -> 320 us under ncu)
#pragma unroll
    for (int extra = 0; extra < kExtraSymbols; ++extra) {
      const uint32_t e2 = tab[tac + (uint32_t)(acc >> (64 - kJpegFastBits))];
      const bool ok = (e2 & kFastFull) && kk < 64 && !bad && nb >= kJpegFastBits;
      const int l2 = ok ? (int)((e2 >> 25) & 31) : 0, adv2 = ok ? (int)((e2 >> kFastAdvShift) & kFastAdvMask) : 0;
      acc <<= l2;
      nb -= l2;
      const int v2 = (int)(int16_t)(e2 & 0xFFFF), pos2 = kk + adv2 - 1;
      if (ok && v2 != 0) myblk[min(pos2, 63)] = (int16_t)v2;
      kk += adv2;
    }
    if (kk >= 64 || bad) {                           // block done: blocks are stored in decode order
      // one bulk copy of the 128-byte block (the generic-proxy coefficient stores made
      // visible to the async proxy first); the block is re-zeroed once it has been read
      uint4* z = reinterpret_cast<uint4*>(myblk);
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(myblk);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(cb), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 8; ++j) z[j] = make_uint4(0, 0, 0, 0);
      cb += 64;
      kk = 0;
      if (++b == bpm) { b = 0; ++m; }
      if (bad || m >= m1) {
        if (bad) { A.status[s].value = k; A.status[s].kind = JST_BAD_CODE; }
        active = false;
      } else {
        comp_tables();
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // this thread's block stores complete
}

// ------------------------------------------------------------------- J3
// Dequantize + islow IDCT (13-bit constants, 2 pass-1 bits, 32-bit modular
// arithmetic as oracle/jpeg_oracle.c) of one 8x8 block in registers.

// four s32 -> u8 with saturation, packed little-endian p0 p1 p2 p3 (two cvt.pack.sat)
__device__ __forceinline__ uint32_t pack4_sat(int p0, int p1, int p2, int p3) {
  uint32_t t, d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(t) : "r"(p3), "r"(p2));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(p1), "r"(p0), "r"(t));
  return d;
}
__device__ __forceinline__ uint32_t range_out(int v) {   // post-IDCT range_limit[v & 1023]
  int s = ((v & 1023) ^ 512) - 512 + 128;
  return (uint32_t)min(max(s, 0), 255);
}

template <bool kPass1>
__device__ __forceinline__ void idct_1d(int& x0, int& x1, int& x2, int& x3, int& x4, int& x5, int& x6, int& x7) {
  // 32-bit modular arithmetic, exactly oracle/jpeg_oracle.c idct_pass
  constexpr int CB = 13, P1 = 2, SH = kPass1 ? CB - P1 : CB + P1 + 3;
  constexpr uint32_t RND = 1u << (SH - 1);
  uint32_t z1, z2, z3, z4, z5, t0, t1, t2, t3, t10, t11, t12, t13;
  z2 = (uint32_t)x2; z3 = (uint32_t)x6;
  z1 = (z2 + z3) * 4433u;
  t2 = z1 + z3 * (uint32_t)-15137;
  t3 = z1 + z2 * 6270u;
  t0 = ((uint32_t)x0 + (uint32_t)x4) << CB;
  t1 = ((uint32_t)x0 - (uint32_t)x4) << CB;
  t10 = t0 + t3; t13 = t0 - t3; t11 = t1 + t2; t12 = t1 - t2;
  t0 = (uint32_t)x7; t1 = (uint32_t)x5; t2 = (uint32_t)x3; t3 = (uint32_t)x1;
  z1 = t0 + t3; z2 = t1 + t2; z3 = t0 + t2; z4 = t1 + t3;
  z5 = (z3 + z4) * 9633u;
  t0 *= 2446u; t1 *= 16819u; t2 *= 25172u; t3 *= 12299u;
  z1 *= (uint32_t)-7373; z2 *= (uint32_t)-20995; z3 *= (uint32_t)-16069; z4 *= (uint32_t)-3196;
  z3 += z5; z4 += z5;
  t0 += z1 + z3; t1 += z2 + z4; t2 += z2 + z3; t3 += z1 + z4;
  x0 = (int)(t10 + t3 + RND) >> SH; x7 = (int)(t10 - t3 + RND) >> SH;
  x1 = (int)(t11 + t2 + RND) >> SH; x6 = (int)(t11 - t2 + RND) >> SH;
  x2 = (int)(t12 + t1 + RND) >> SH; x5 = (int)(t12 - t1 + RND) >> SH;
  x3 = (int)(t13 + t0 + RND) >> SH; x4 = (int)(t13 - t0 + RND) >> SH;
}

// One block: coefficients (global, zig-zag order as J2 stores them) -> 8 rows
// of 8 bytes at dst (stride bytes).  The de-zigzag is a compile-time register
// permutation; the quant table is in natural order.
__device__ __forceinline__ void idct_block(const int16_t* coef, const uint16_t* q, uint8_t* dst, int stride) {
  constexpr uint8_t kNat[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
  const uint4* src = reinterpret_cast<const uint4*>(coef);
  const uint4* q4 = reinterpret_cast<const uint4*>(q);
  uint32_t cw[32], qw[32];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint4 cv = __ldg(src + r), qv = __ldg(q4 + r);   // L1-allocating: the 8 loads share 4 lines
    cw[4 * r] = cv.x; cw[4 * r + 1] = cv.y; cw[4 * r + 2] = cv.z; cw[4 * r + 3] = cv.w;
    qw[4 * r] = qv.x; qw[4 * r + 1] = qv.y; qw[4 * r + 2] = qv.z; qw[4 * r + 3] = qv.w;
  }
  int w[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) {
    const int n = kNat[k];
    const int c = (int)(int16_t)((k & 1) ? cw[k >> 1] >> 16 : cw[k >> 1] & 0xFFFF);
    const uint32_t qq = (n & 1) ? qw[n >> 1] >> 16 : qw[n >> 1] & 0xFFFF;
    w[n] = (int)((uint32_t)c * qq);
  }
#pragma unroll
  for (int col = 0; col < 8; ++col) {
    int* x = w + col;
    if ((x[8] | x[16] | x[24] | x[32] | x[40] | x[48] | x[56]) == 0) {
      const int dc = (int)((uint32_t)x[0] << 2);
#pragma unroll
      for (int r = 0; r < 8; ++r) x[r * 8] = dc;
    } else {
      idct_1d<true>(x[0], x[8], x[16], x[24], x[32], x[40], x[48], x[56]);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int* x = w + r * 8;
    uint2 row;
    if ((x[1] | x[2] | x[3] | x[4] | x[5] | x[6] | x[7]) == 0) {
      const uint32_t v = range_out((int)((uint32_t)x[0] + 16u) >> 5);
      row.x = row.y = v * 0x01010101u;
    } else {
      idct_1d<false>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
      // range_limit[v & 1023] = clamp(((v & 1023) ^ 512) - 512 + 128, 0, 255): the clamp is
      // the saturation of the byte packing
      int q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = ((x[j] & 1023) ^ 512) - 384;
      row = make_uint2(pack4_sat(q[0], q[1], q[2], q[3]), pack4_sat(q[4], q[5], q[6], q[7]));
    }
    *reinterpret_cast<uint2*>(dst + (size_t)r * stride) = row;
  }
}

// J3: thread per block, blocks taken in the coefficient buffer's MCU order.
constexpr int kIdctThreads = 128;

__global__ void __launch_bounds__(kIdctThreads) jpeg_idct_kernel(const JpegArgs A) {
  // grid (block chunks of the largest sample, samples): no search for the sample
  const int s = blockIdx.y;
  const JpegDesc& J = A.jd[s];
  const uint32_t rel = blockIdx.x * kIdctThreads + threadIdx.x;
  if (rel >= J.n_blocks || J.n_int == 0 || A.status[s].kind != 0) return;
  const uint64_t g = J.blk_base + rel;
  const uint32_t bpm = J.bpm;
  const uint32_t m = rel / bpm, b = rel - m * bpm;
  const uint32_t e = (uint32_t)(J.sched >> (4 * b)) & 15u, c = e & 3;
  const JComp& C = J.comp[c];
  const uint32_t my = m / J.mcus_x, mx = m - my * J.mcus_x;
  const uint32_t V = J.ncomp == 1 ? 1 : C.v, H = J.ncomp == 1 ? 1 : C.h;
  const uint32_t by = my * V + ((e >> 2) & 1), bx = mx * H + (e >> 3), pw = (uint32_t)C.bw * 8;
  if (!jpeg_block_needed(J, (int)c, (int)by, (int)bx)) return;
  uint8_t* plane = A.planes + (J.blk_base + J.plane_blk[c]) * 64;
  idct_block(A.coef + g * 64, A.quant[C.q].q, plane + (size_t)by * 8 * pw + bx * 8, (int)pw);
}

// J4: thread per 4 output pixels of one row.  libjpeg's fancy upsampling
// (h2v1 / h1v2 / h2v2 triangle filters with edge replication; box when the
// downsampled width is <= 2) and JFIF YCbCr -> RGB in 16-bit fixed point.
constexpr int kColorThreads = 256;

struct Plane {
  const uint8_t* p;
  int pw, dw, dh, rh, rv;          // row pitch, downsampled dims, upsampling ratios
};

__device__ __forceinline__ int plane_sample(const Plane& c, int y, int x) {
  auto at = [&](int yy, int xx) { return (int)__ldg(c.p + (size_t)yy * c.pw + xx); };
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

__device__ __forceinline__ uint32_t ycc_r(int Y, int cr) { return (uint32_t)min(max(Y + ((91881 * cr + 32768) >> 16), 0), 255); }
__device__ __forceinline__ uint32_t ycc_g(int Y, int cb, int cr) {
  return (uint32_t)min(max(Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16), 0), 255);
}
__device__ __forceinline__ uint32_t ycc_b(int Y, int cb) { return (uint32_t)min(max(Y + ((116130 * cb + 32768) >> 16), 0), 255); }
__device__ __forceinline__ int ycc_r_raw(int Y, int cr) { return Y + ((91881 * cr + 32768) >> 16); }
__device__ __forceinline__ int ycc_g_raw(int Y, int cb, int cr) { return Y + ((-22554 * cb + 32768 - 46802 * cr) >> 16); }
__device__ __forceinline__ int ycc_b_raw(int Y, int cb) { return Y + ((116130 * cb + 32768) >> 16); }

template <int N>
__device__ __forceinline__ void store_px(uint8_t* o, const uint32_t (&px)[N], int n) {   // first n bytes, packed
  const uintptr_t a = reinterpret_cast<uintptr_t>(o);
  if (n == N && (a & 7) == 0 && (N & 7) == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 8)
      *reinterpret_cast<uint2*>(o + k) =
          make_uint2(px[k] | px[k + 1] << 8 | px[k + 2] << 16 | px[k + 3] << 24,
                     px[k + 4] | px[k + 5] << 8 | px[k + 6] << 16 | px[k + 7] << 24);
  } else if (n == N && (a & 3) == 0 && (N & 3) == 0) {
#pragma unroll
    for (int k = 0; k < N; k += 4)
      *reinterpret_cast<uint32_t*>(o + k) = px[k] | px[k + 1] << 8 | px[k + 2] << 16 | px[k + 3] << 24;
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) if (k < n) o[k] = (uint8_t)px[k];
  }
}

// J4: CTA per (sample, band of kColorRows rows); a thread produces 8 output
// pixels of one row per step (4:2:0 fast path: one 8-byte luma load and, per
// chroma plane and row, one 4-byte load plus the two edge-clamped
// neighbours); any other layout goes per pixel through plane_sample.
constexpr int kColorRows = 64;

__global__ void __launch_bounds__(kColorThreads) jpeg_color_kernel(const JpegArgs A) {
  const int s = blockIdx.y;
  __shared__ Plane sP[3];
  __shared__ int s_ok, s_fast;
  const JpegDesc& J = A.jd[s];
  const SampleDesc* d = sdesc(A, s);
  const int w = d->w, nc = J.ncomp;
  const int y_lo = max((int)blockIdx.x * kColorRows, (int)J.win[0]);
  const int y_hi = min((int)(blockIdx.x + 1) * kColorRows, (int)J.win[1]);
  if (threadIdx.x < 3) {                            // one lane per component (independent loads)
    const int c = threadIdx.x;
    if (c < nc) {
      const JComp& C = J.comp[c];
      Plane q;
      q.p = A.planes + (J.blk_base + J.plane_blk[c]) * 64;
      q.pw = C.bw * 8; q.dw = C.dw; q.dh = C.dh; q.rh = J.hmax / C.h; q.rv = J.vmax / C.v;
      sP[c] = q;
    }
    if (c == 0) s_ok = J.n_int != 0 && A.status[s].kind == 0 && y_lo < y_hi && J.win[2] < J.win[3];
  }
  __syncwarp();
  if (threadIdx.x == 0)
    s_fast = nc == 3 && sP[0].rh == 1 && sP[0].rv == 1 && sP[1].rh == 2 && sP[1].rv == 2 && sP[2].rh == 2 &&
             sP[2].rv == 2 && sP[1].dw > 2 && sP[2].dw > 2 && sP[1].dw == sP[2].dw && sP[1].dh == sP[2].dh &&
             sP[1].pw == sP[2].pw;
  __syncthreads();
  if (!s_ok) return;
  // octets covering the window's columns (their extra pixels lie inside the decoded MCUs)
  const int q_lo = J.win[2] >> 3, no = ((J.win[3] + 7) >> 3) - q_lo, n = (y_hi - y_lo) * no;
  uint8_t* const out = A.scratch + (size_t)s * A.scratch_bytes;
  const size_t pitch = A.exact_pitch ? (size_t)w * nc : (size_t)jpeg_scratch_pitch(w, nc);
  if (nc == 1) {
    const Plane P0 = sP[0];
    for (int t = threadIdx.x; t < n; t += kColorThreads) {
      const int yy = t / no, q = t - yy * no + q_lo, y = y_lo + yy, x0 = 8 * q;
      uint32_t px[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) px[k] = (uint32_t)plane_sample(P0, y, min(x0 + k, w - 1));
      store_px(out + (size_t)y * pitch + x0, px, min(8, w - x0));
    }
    return;
  }
  if (s_fast) {                                      // 4:2:0 fancy (h2v2)
    const uint8_t* yp = sP[0].p;
    const uint8_t* cbp = sP[1].p;
    const uint8_t* crp = sP[2].p;
    const int ypw = sP[0].pw, cpw = sP[1].pw, dw = sP[1].dw, dh = sP[1].dh;
    const int lane = threadIdx.x & 31;
    // item t = (row yy, octet q): consecutive threads take consecutive octets of a
    // row, so a chroma word's edge neighbours come from the adjacent lanes
    int yy = threadIdx.x / no, qq = threadIdx.x - yy * no;
    const int dyy = kColorThreads / no, dqq = kColorThreads - dyy * no;
    for (int t = threadIdx.x; __any_sync(0xffffffffu, t < n); t += kColorThreads) {
      const bool act = t < n;
      const int q = qq + q_lo, y = y_lo + yy, x0 = 8 * q;
      const int i = y >> 1, i1 = (y & 1) ? min(i + 1, dh - 1) : max(i - 1, 0), j0 = 4 * q;
      const int ja = max(j0 - 1, 0), je = min(j0 + 4, dw - 1);
      const bool whole = j0 + 4 <= dw;
      uint2 y8 = make_uint2(0, 0);
      uint32_t w4[4] = {0, 0, 0, 0};                 // Cb row i, Cb row i1, Cr row i, Cr row i1 (bytes j0 .. j0+3)
      if (act) {
        y8 = __ldg(reinterpret_cast<const uint2*>(yp + (size_t)y * ypw + x0));
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const uint8_t* ra = (c ? crp : cbp) + (size_t)i * cpw;
          const uint8_t* rb = (c ? crp : cbp) + (size_t)i1 * cpw;
          if (whole) {
            w4[2 * c] = __ldg(reinterpret_cast<const uint32_t*>(ra + j0));
            w4[2 * c + 1] = __ldg(reinterpret_cast<const uint32_t*>(rb + j0));
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int jj = min(j0 + k, dw - 1);
              w4[2 * c] |= (uint32_t)__ldg(ra + jj) << (8 * k);
              w4[2 * c + 1] |= (uint32_t)__ldg(rb + jj) << (8 * k);
            }
          }
        }
      }
      // neighbours' words: lane - 1 holds octet q - 1 of the same row when tl == t - 1 etc.
      const int tl = __shfl_up_sync(0xffffffffu, t, 1), tr = __shfl_down_sync(0xffffffffu, t, 1);
      uint32_t wl[4], wr[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        wl[k] = __shfl_up_sync(0xffffffffu, w4[k], 1);
        wr[k] = __shfl_down_sync(0xffffffffu, w4[k], 1);
      }
      if (!act) { yy += dyy; qq += dqq; if (qq >= no) { qq -= no; ++yy; } continue; }
      const bool left_ok = lane > 0 && tl == t - 1 && qq > 0, right_ok = lane < 31 && tr == t + 1 && qq + 1 < no && whole;
      int u[2][8];
#pragma unroll
      for (int c = 0; c < 2; ++c) {                  // chroma columns j0-1 .. j0+4 (edge-clamped)
        const uint8_t* ra = (c ? crp : cbp) + (size_t)i * cpw;
        const uint8_t* rb = (c ? crp : cbp) + (size_t)i1 * cpw;
        const uint32_t a4 = w4[2 * c], b4 = w4[2 * c + 1];
        int cs[6];
        if (j0 == 0) cs[0] = 3 * (int)(a4 & 0xFF) + (int)(b4 & 0xFF);
        else if (left_ok) cs[0] = 3 * (int)(wl[2 * c] >> 24) + (int)(wl[2 * c + 1] >> 24);
        else cs[0] = 3 * __ldg(ra + ja) + __ldg(rb + ja);
        if (right_ok && j0 + 4 < dw) cs[5] = 3 * (int)(wr[2 * c] & 0xFF) + (int)(wr[2 * c + 1] & 0xFF);
        else cs[5] = 3 * __ldg(ra + je) + __ldg(rb + je);
#pragma unroll
        for (int k = 0; k < 4; ++k) cs[1 + k] = 3 * (int)((a4 >> (8 * k)) & 0xFF) + (int)((b4 >> (8 * k)) & 0xFF);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          u[c][2 * k] = ((3 * cs[1 + k] + cs[k] + 8) >> 4) - 128;
          u[c][2 * k + 1] = ((3 * cs[1 + k] + cs[2 + k] + 7) >> 4) - 128;
        }
      }
      // R, G, B unclamped; the clamp to [0, 255] is the saturation of the byte packing
      int v[24];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int Y = (int)(((k < 4 ? y8.x : y8.y) >> (8 * (k & 3))) & 0xFF), cb = u[0][k], cr = u[1][k];
        v[3 * k] = ycc_r_raw(Y, cr); v[3 * k + 1] = ycc_g_raw(Y, cb, cr); v[3 * k + 2] = ycc_b_raw(Y, cb);
      }
      uint8_t* const o = out + (size_t)y * pitch + (size_t)x0 * 3;
      if (x0 + 8 <= w && (reinterpret_cast<uintptr_t>(o) & 7) == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
          *reinterpret_cast<uint2*>(o + 8 * q) = make_uint2(pack4_sat(v[8 * q], v[8 * q + 1], v[8 * q + 2], v[8 * q + 3]),
                                                            pack4_sat(v[8 * q + 4], v[8 * q + 5], v[8 * q + 6], v[8 * q + 7]));
      } else {
        uint32_t px[24];
#pragma unroll
        for (int i = 0; i < 24; ++i) px[i] = (uint32_t)min(max(v[i], 0), 255);
        store_px(o, px, 3 * min(8, w - x0));
      }
      yy += dyy; qq += dqq; if (qq >= no) { qq -= no; ++yy; }
    }
    return;
  }
  const Plane P0 = sP[0], P1 = sP[1], P2 = sP[2];
  for (int t = threadIdx.x; t < n; t += kColorThreads) {
    const int yy = t / no, q = t - yy * no + q_lo, y = y_lo + yy, x0 = 8 * q;
    uint32_t px[24];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int x = min(x0 + k, w - 1);
      const int Y = plane_sample(P0, y, x), cb = plane_sample(P1, y, x) - 128, cr = plane_sample(P2, y, x) - 128;
      px[3 * k] = ycc_r(Y, cr); px[3 * k + 1] = ycc_g(Y, cb, cr); px[3 * k + 2] = ycc_b(Y, cb);
    }
    store_px(out + (size_t)y * pitch + (size_t)x0 * 3, px, 3 * min(8, w - x0));
  }
}

static int sm_count() {                     // of the current device (cached per device)
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] > 0 ? cache[dev] : 148;
}

int launch_jpeg(const JpegArgs& A, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (A.count <= 0 || A.total_int == 0) return 0;
  const bool smem = A.n_huff <= kJpegSmemTables;
  const int hsmem = huff_blk_bytes() +
                    (smem ? A.n_huff * (int)sizeof(JHuff::fast) + (A.n_huff * (10 * 4 + 256) + 15) / 16 * 16 : 0);
  // a thread per restart interval, CTAs of kHuffThreads consecutive intervals
  const unsigned hgrid = (unsigned)(((uint64_t)A.total_int + kHuffThreads - 1) / kHuffThreads);
  if (smem) {
    cudaFuncSetAttribute(jpeg_huffman_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem);
    cudaFuncSetAttribute(jpeg_huffman_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    jpeg_huffman_kernel<true><<<hgrid, kHuffThreads, hsmem, st>>>(A);
  } else {
    cudaFuncSetAttribute(jpeg_huffman_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem);
    jpeg_huffman_kernel<false><<<hgrid, kHuffThreads, hsmem, st>>>(A);
  }
  jpeg_idct_kernel<<<dim3((A.max_blocks + kIdctThreads - 1) / kIdctThreads, A.count), kIdctThreads, 0, st>>>(A);
  jpeg_color_kernel<<<dim3((A.max_quads + kColorRows - 1) / kColorRows, A.count), kColorThreads, 0, st>>>(A);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace bbx
