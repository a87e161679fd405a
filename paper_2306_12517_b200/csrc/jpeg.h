// JPEG codec (codec id 3): host header parse + device decoder.  Shared by
// jpeg_host.cpp (parse, table build), jpeg.cu (kernels) and engine.cpp.
//
// Host (jpeg_prepare, once per sample, cached): header parse, and a scan of
// the entropy-coded segment for its RSTn markers (T.81 B.2.5) -- count and
// sequence checked, each restart interval's first byte recorded.
// Device pipeline for the JPEG samples of one batch:
//   J2 jpeg_huffman_kernel   thread per restart interval, reading the stuffed
//                            bytes directly (0xFF00 -> 0xFF, marker -> zeros,
//                            T.81 F.1.2.3): one flat loop, up to five symbols
//                            per iteration (T.81 F.2.2), shared-memory tables
//                            that resolve code + extra bits in one lookup;
//                            coefficients stored as int16[64] in zig-zag order
//   J3 jpeg_idct_kernel      thread per 8x8 block: dequantize + islow IDCT in
//                            registers -> u8 component planes
//   J4 jpeg_color_kernel     thread per 8 output pixels: fancy chroma
//                            upsampling + YCbCr->RGB into the sample's decode
//                            scratch, which K1 reads like an RLE-expanded image
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define BBX_HD __host__ __device__
#else
#define BBX_HD
#endif

namespace bbx {

constexpr int kJpegFastBits = 11;         // Huffman lookahead bits (fast table)
constexpr int kJpegMaxHuff = 512;         // device Huffman table pool entries
constexpr int kJpegMaxQuant = 256;        // device quant table pool entries
constexpr int kJpegSmemTables = 8;        // J2 stages the pool in smem when it holds at most this many

// Fast-table entry (u32) indexed by the next kJpegFastBits bits of the stream:
//   bit 31 valid (code <= kJpegFastBits bits; else the maxcode search),
//   bit 30 full: code + extra bits fit, bits 0..15 hold the decoded value
//          (EXTENDed coefficient, or the DC difference); not full: bits 0..3
//          hold the extra bits still to read,
//   bits 25..29 bits to consume (full: code + extra; else the code only),
//   bits 16..22 zig-zag advance: run + 1 (1 for DC), 64 for end of block
//          (AC size 0, run < 15) -- the coefficient lands at k + advance - 1
constexpr uint32_t kFastValid = 1u << 31, kFastFull = 1u << 30;
constexpr int kFastAdvShift = 16;
constexpr uint32_t kFastAdvMask = 127u;

struct JHuff {                            // one Huffman table, device form
  uint32_t fast[1 << kJpegFastBits];
  int32_t maxcode[18];                    // largest code of each length, -1 if none; [17] sentinel
  int32_t valoff[18];                     // vals index = code + valoff[len]
  uint8_t vals[256];
  int32_t is_ac, pad[3];
};
struct JQuant { uint16_t q[64]; };        // natural order

struct JComp {
  uint16_t dc, ac, q;                     // table pool ids
  uint8_t h, v;                           // sampling factors (1 or 2; 1 for single-component files)
  uint16_t bw, bh;                        // coded blocks per row / column
  uint16_t dw, dh;                        // downsampled width / height (jdsample edge rule)
  uint32_t blk_off;                       // offset of this component's first block inside an MCU
};
static_assert(sizeof(JComp) == 20, "JComp layout");

struct JpegDesc {                         // per sample, staged with the descriptors
  uint32_t scan_off;                      // entropy-coded data start (payload-relative)
  uint32_t scan_end;                      // payload length
  uint16_t mcus_x, mcus_y;
  uint32_t restart;                       // MCUs per interval (all MCUs when no DRI)
  uint8_t ncomp, hmax, vmax, bpm;         // bpm: blocks per MCU
  uint32_t n_int;                         // restart intervals (0: not a JPEG sample)
  uint32_t int_base;                      // first interval in the batch interval table
  uint32_t n_blocks;
  uint64_t blk_base;                      // first block in the batch coefficient buffer (MCU order:
                                          // block b of MCU m at blk_base + m * bpm + b)
  uint64_t reserved;
  uint64_t sched;                         // MCU block b: comp bits 4b..4b+1, v bit 4b+2, h bit 4b+3
  JComp comp[3];
  uint32_t plane_blk[3];                  // component c's pixel plane starts plane_blk[c] blocks into the sample's planes
  uint16_t win[4];                        // pixels the chain reads: rows [win[0], win[1]) x cols [win[2], win[3])
};
static_assert(sizeof(JpegDesc) == 136, "JpegDesc layout");

// Region of interest.  Component c's samples the chain needs: the window's rows
// / columns scaled to the component (plus one on each side when it is
// upsampled 2x: fancy upsampling reads the neighbouring row / column), i.e.
// blocks [lo / 8, hi / 8] of that component.  Restart intervals whose MCUs hold
// none of them are not decoded (DC predictors restart per interval, so nothing
// else depends on them), and their blocks are not inverse-DCT'd.
struct CompSpan { int lo, hi; };                 // inclusive sample range, lo > hi: empty
BBX_HD inline CompSpan jpeg_comp_span(int p0, int p1, int f, int fmax, int dn) {
  CompSpan r{0, -1};
  if (p0 >= p1) return r;
  const int up = fmax / f == 2 ? 1 : 0;
  r.lo = (p0 * f) / fmax - up; if (r.lo < 0) r.lo = 0;
  r.hi = ((p1 - 1) * f) / fmax + up; if (r.hi > dn - 1) r.hi = dn - 1;
  return r;
}
// block (by, bx) of component c needed?
BBX_HD inline bool jpeg_block_needed(const JpegDesc& J, int c, int by, int bx) {
  const JComp& C = J.comp[c];
  const int v = J.ncomp == 1 ? 1 : C.v, h = J.ncomp == 1 ? 1 : C.h;
  const int vm = J.ncomp == 1 ? 1 : J.vmax, hm = J.ncomp == 1 ? 1 : J.hmax;
  const CompSpan ys = jpeg_comp_span(J.win[0], J.win[1], v, vm, C.dh), xs = jpeg_comp_span(J.win[2], J.win[3], h, hm, C.dw);
  return by >= ys.lo / 8 && by <= ys.hi / 8 && bx >= xs.lo / 8 && bx <= xs.hi / 8;
}
struct McuRect { int x0, x1, y0, y1; };          // half-open MCU ranges
BBX_HD inline McuRect jpeg_mcu_rect(const JpegDesc& J) {
  McuRect r{1 << 30, 0, 1 << 30, 0};
  for (int c = 0; c < J.ncomp; ++c) {
    const JComp& C = J.comp[c];
    const int v = J.ncomp == 1 ? 1 : C.v, h = J.ncomp == 1 ? 1 : C.h;
    const int vm = J.ncomp == 1 ? 1 : J.vmax, hm = J.ncomp == 1 ? 1 : J.hmax;
    const CompSpan ys = jpeg_comp_span(J.win[0], J.win[1], v, vm, C.dh), xs = jpeg_comp_span(J.win[2], J.win[3], h, hm, C.dw);
    if (ys.lo > ys.hi || xs.lo > xs.hi) continue;
    const int y0 = ys.lo / (8 * v), y1 = ys.hi / (8 * v) + 1, x0 = xs.lo / (8 * h), x1 = xs.hi / (8 * h) + 1;
    if (y0 < r.y0) r.y0 = y0;
    if (y1 > r.y1) r.y1 = y1;
    if (x0 < r.x0) r.x0 = x0;
    if (x1 > r.x1) r.x1 = x1;
  }
  if (r.y0 >= r.y1 || r.x0 >= r.x1) r = McuRect{0, 0, 0, 0};
  return r;
}

// Restart interval k of a sample holds MCUs of the region of interest?  (DC
// predictors restart per interval, so intervals outside it are never decoded;
// conservative across MCU-row wraps.)
BBX_HD inline bool jpeg_interval_live(const JpegDesc& J, const McuRect& R, uint32_t k) {
  const uint32_t total = (uint32_t)J.mcus_x * J.mcus_y, m = k * J.restart;
  const uint32_t m1 = m + J.restart < total ? m + J.restart : total;
  if (m >= m1) return false;
  const uint32_t mx = J.mcus_x, ra = m / mx, rb = (m1 - 1) / mx;
  if ((int)rb < R.y0 || (int)ra >= R.y1) return false;
  if (ra == rb && ((int)((m1 - 1) % mx) < R.x0 || (int)(m % mx) >= R.x1)) return false;
  return true;
}

// Per-sample status kind written by J2 (SampleStatus::kind).
enum : int32_t { JST_BAD_CODE = 3 };

// Everything the JPEG kernels need for one batch of one plan.
struct JpegArgs {
  const uint8_t* desc;                    // SampleDesc array (desc_stride apart)
  int32_t desc_stride;
  const uint8_t* payload;                 // payload base (staged region or resident heap)
  const JpegDesc* jd;                     // count entries
  const uint32_t* int_prefix;             // count + 1: exclusive prefix of n_int
  const uint64_t* blk_prefix;             // count + 1: exclusive prefix of n_blocks
  uint8_t* planes;                        // total blocks x 64: component planes (J3 -> J4)
  const uint32_t* starts;                 // per interval: first entropy-coded byte (payload-relative, host scan)
  int16_t* coef;                          // total blocks x 64
  uint8_t* scratch;                       // count x scratch_bytes: decoded HWC u8
  int64_t scratch_bytes;
  int32_t exact_pitch;                    // 1: rows w*c bytes apart; 0: jpeg_scratch_pitch (16-B aligned rows)
  const JHuff* huff;                      // table pools
  const JQuant* quant;
  int32_t n_huff;                         // pool entries in use
  int32_t coef_zeroed;                    // coef holds zeros where J2 stores nothing
  struct SampleStatus* status;
  int32_t count;
  uint32_t total_int;
  uint64_t total_blocks;
  int32_t max_quads;                      // largest image height in the batch (J4 grid: bands of rows)
  uint32_t max_blocks;                    // most blocks of one sample in the batch (J3 grid)
};

// jpeg.cu
int launch_jpeg(const JpegArgs& A, void* stream);

// jpeg_host.cpp
struct JpegHeader {
  int width = 0, height = 0, ncomp = 0, restart = 0;
  uint32_t scan_off = 0;
  struct Comp { int id, h, v, tq, td, ta; } comp[3];
  // raw tables referenced by the components: DHT (counts[16] + values) / DQT (natural order)
  struct Huff { bool present = false; uint8_t counts[16]; uint8_t vals[256]; int nvals = 0; } dc[4], ac[4];
  struct Quant { bool present = false; uint16_t q[64]; } qt[4];
};
// Parses markers up to SOS.  Returns 0, or fills *err with the reason.
int jpeg_parse_header(const uint8_t* p, uint64_t n, JpegHeader* h, char* err, int errlen);
// Builds the device form of a DHT table; false if it is malformed.
bool jpeg_build_huff(const JpegHeader::Huff& t, bool is_ac, JHuff* out);

}  // namespace bbx
