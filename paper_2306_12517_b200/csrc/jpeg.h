// JPEG codec (codec id 3): host header parse + device decoder.  Shared by
// jpeg_host.cpp (parse, table registry), jpeg.cu (kernels) and engine.cpp.
//
// Device pipeline for the JPEG samples of one batch:
//   J1 jpeg_scan_kernel     warp per sample: RSTn marker search over the
//                           entropy-coded segment -> start/end of every
//                           restart interval (T.81 F.1.2.3 / B.2.5)
//   J2 jpeg_huffman_kernel  thread per restart interval: Huffman decode of
//                           the interval's MCUs (T.81 F.2.2) -> int16
//                           coefficient blocks, natural order
//   J3 jpeg_idct_kernel     thread per block: dequantize + islow IDCT -> u8
//                           component planes
//   J4 jpeg_color_kernel    thread per pixel: fancy chroma upsampling +
//                           YCbCr -> RGB into the sample's decode scratch,
//                           which K1 then reads like an RLE-expanded image
#pragma once
#include <cstdint>

namespace bbx {

constexpr int kJpegLook = 9;              // Huffman lookahead bits (fast table)
constexpr int kJpegMaxHuff = 512;         // device Huffman table pool entries
constexpr int kJpegMaxQuant = 256;        // device quant table pool entries

struct JHuff {                            // one Huffman table, device form
  uint16_t look[1 << kJpegLook];          // (len << 8) | symbol; 0 = code longer than kJpegLook
  int32_t maxcode[18];                    // largest code of each length, -1 if none; [17] sentinel
  int32_t valoff[18];                     // vals index = code + valoff[len]
  uint8_t vals[256];
};
struct JQuant { uint16_t q[64]; };        // natural order

struct JComp {
  uint16_t dc, ac, q;                     // table pool ids
  uint8_t h, v;                           // sampling factors (1 or 2; 1 for single-component files)
  uint16_t bw, bh;                        // coded blocks per row / column
  uint16_t dw, dh;                        // downsampled width / height (jdsample edge rule)
  uint32_t blk_off;                       // first block, relative to the sample's block base
};
static_assert(sizeof(JComp) == 20, "JComp layout");

struct JpegDesc {                         // per sample, staged with the descriptors
  uint32_t scan_off;                      // entropy-coded data start (payload-relative)
  uint32_t scan_end;                      // payload length
  uint16_t mcus_x, mcus_y;
  uint32_t restart;                       // MCUs per interval (all MCUs when no DRI)
  uint8_t ncomp, hmax, vmax, pad0;
  uint32_t n_int;                         // restart intervals (0: not a JPEG sample)
  uint32_t int_base;                      // first interval in the batch interval table
  uint32_t n_blocks;
  uint64_t blk_base;                      // first block in the batch coefficient / plane buffers
  JComp comp[3];
  uint32_t pad1[3];
};
static_assert(sizeof(JpegDesc) == 112, "JpegDesc layout");

// Per-sample status kinds written by J1/J2 (SampleStatus::kind).
enum : int32_t { JST_BAD_CODE = 3, JST_MARKER_COUNT = 4, JST_MARKER_SEQ = 5 };

// Everything the JPEG kernels need for one batch of one plan.
struct JpegArgs {
  const uint8_t* desc;                    // SampleDesc array (P.desc_stride apart)
  int32_t desc_stride;
  const uint8_t* payload;                 // payload base (staged region or resident heap)
  const JpegDesc* jd;                     // count entries
  const uint32_t* int_prefix;             // count + 1: exclusive prefix of n_int
  const uint64_t* blk_prefix;             // count + 1: exclusive prefix of n_blocks
  uint32_t* istart;                       // interval tables (total intervals)
  uint32_t* iend;
  int16_t* coef;                          // total blocks x 64
  uint8_t* planes;                        // total blocks x 64 (component planes)
  uint8_t* scratch;                       // count x scratch_bytes: decoded HWC u8
  int64_t scratch_bytes;
  const JHuff* huff;                      // table pools
  const JQuant* quant;
  struct SampleStatus* status;
  int32_t count;
  uint32_t total_int;
  uint64_t total_blocks;
  int32_t max_pixels;                     // largest h*w in the batch
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
bool jpeg_build_huff(const JpegHeader::Huff& t, JHuff* out);

}  // namespace bbx
