// Internal structures shared by the host engine (engine.cpp) and the sm_100a
// kernels (kernels.cu).  See DESIGN.md §3 for the HBM layout they describe.
#pragma once
#include <cstdint>
#include <cstddef>

#include "../../include/bbx.h"

namespace bbx {

enum SrcKind : int32_t { SRC_DECODE = 0, SRC_RESAMPLE = 1, SRC_ARRAY = 2 };
enum Codec : int32_t { CODEC_RAW = 0, CODEC_RLE = 1, CODEC_SUB2 = 2, CODEC_JPEG = 3 };
enum ValueMode : int32_t { VAL_COPY = 0, VAL_FMA = 1, VAL_DIRECT = 2, VAL_LUT = 3 };

constexpr int kMaxRemaps = 12;
constexpr int kMaxValueOps = 8;
constexpr int kDescHeader = 32;     // bytes before the per-sample params
// column-walker K1 compile-time shape (the defaults are the measured best;
// _build.build(defines=...) makes A/B builds for measurement scripts)
#ifndef BBX_CW_STAGES
#define BBX_CW_STAGES 2
#endif
#ifndef BBX_CW_ROWS
#define BBX_CW_ROWS 16
#endif
#ifndef BBX_CW_RUN
#define BBX_CW_RUN 3
#endif
constexpr int kCwStages = BBX_CW_STAGES;   // source-row pipeline stages
constexpr int kCwRows = BBX_CW_ROWS;       // output rows per tile (fewer when a tile would span > 32 source rows)
constexpr int kCwRun = BBX_CW_RUN;         // consecutive tiles per ticket
constexpr int kThreads = 256;       // CTA size of the image kernels
constexpr int kStreams = 2;         // compute streams a loader alternates its batches between (A/B, configs[2]:
                                    // 3 streams +3 % value but -20 % e2e, 4 streams slower on both)
constexpr int kSmemTarget = 56 * 1024;   // 4 CTAs of 256 threads per SM
constexpr int kSmemBudget = 200 * 1024;

// One geometric op after the source, in chain order.  Separable by axis:
// output (y, x) -> input (fy(y), fx(x)).
struct Remap {
  int32_t kind;          // BBX_OP_CROP / BBX_OP_FLIP / BBX_OP_RESIZE
  int32_t in_h, in_w;    // input spec (pipeline.py output_spec propagation)
  int32_t out_h, out_w;
  int32_t prm;           // first per-sample param slot (crop: top, left; flip: bit)
};

// Shared-memory layout of K1 for one plan (computed once on the host).
struct SmemLayout {
  int32_t nslot;        // staged source rows (R nearest, 2R bilinear)
  int32_t span_pad;     // bytes per staged source row
  int32_t hrow_pad;     // bytes per horizontally-resampled row
  int32_t xt_off, meta_off, src_off, h_off, total;
};

// Everything the kernels need about one compiled chain; passed by value.
struct PlanDev {
  int32_t src_kind;
  int32_t canvas_h, canvas_w, channels;   // source op output (Decode: max dims)
  int32_t src_row_w;                       // widest source image row in pixels (field max width)
  int32_t src_elem;                        // bytes per source element (1 for images)
  int32_t src_dtype;                       // bbx_dtype of the source elements
  int32_t out_h, out_w, out_c;             // final output (3-D view; arrays: 1 x N x 1)
  int32_t out_dtype;
  int32_t n_remaps;
  Remap remaps[kMaxRemaps];
  int32_t value_mode;
  int32_t n_vops;
  // normalize ops only (ToFloat is implicit); scalar Normalize is replicated over [4]
  float vop_mean[kMaxValueOps][4];
  float vop_std[kMaxValueOps][4];
  float vop_inv[kMaxValueOps][4];          // RN(1/std), for VAL_FMA
  int32_t desc_stride;
  int32_t n_params;
  int32_t rows_per_tile;
  int32_t tiles_per_sample;
  int64_t out_sample_elems;
  int64_t scratch_bytes;                   // per-sample decode scratch (RLE)
  int32_t has_remaps_3d;                   // arrays: 3-D remaps present
  int32_t smem_bytes;
  int32_t lin32;                           // bilinear axis math fits 32-bit
  uint32_t ow_magic, gpr_magic;            // ceil(2^32/d) fast-division constants, 0 = use /
  uint32_t linx_magic, liny_magic;         // for 2*canvas_w / 2*canvas_h (bilinear axes), 0 = use /
  int32_t h_tpc;                           // horizontal pass: threads per output column
  int32_t tab_stride;                      // K1 prologue table words per sample
  // column-walker K1 (bilinear, 3 channels): a compute thread owns two output
  // columns of every tile its CTA takes (image_kernel.cuh, image_cw_kernel)
  int32_t cw, cw_smem, cw_npair;
  int32_t cw_warps;                        // compute warps per CTA (plus one copy-issuing warp)
  int32_t cw_slots;                        // source rows one pipeline stage holds (<= 32)
  int32_t cw_run;                          // consecutive tiles a CTA takes per ticket
  int32_t cw_affine;                       // f16/bf16 values as fma(u, cw_aff_a[c], cw_aff_b[c]) (host-proven exact)
  float cw_aff_a[4], cw_aff_b[4];
  // the same maps as the f32 pairs a compute thread's packed values use: channels (0,1) (2,0) (1,2)
  alignas(8) float cw_pair_a[6];
  alignas(8) float cw_pair_b[6];
  SmemLayout lay;
};

// Row pitch of a JPEG sample's decoded (HWC u8) scratch image: 16-byte aligned
// rows, so J4 stores whole 8-byte words and K1 bulk-copies from aligned rows.
#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t jpeg_scratch_pitch(int w, int c) { return ((int64_t)w * c + 15) / 16 * 16; }

// Per-sample descriptor header (kDescHeader bytes), followed by n_params int32.
struct SampleDesc {
  uint64_t src;    // payload byte offset from the launch's payload base
  uint32_t len;    // payload length
  uint16_t h, w;   // image cell dims
  uint8_t c, codec, skip, flags;  // flags bit0: staged payload is a window (RAW only)
  int32_t index_lo;  // sample index (low 32 bits, diagnostics)
  uint32_t wstride;  // windowed: bytes per staged row
  uint16_t wy0, wx0; // windowed: image coordinates of the window's first row / column
};
constexpr uint8_t kDescWindowed = 1;
static_assert(sizeof(SampleDesc) == kDescHeader, "descriptor header layout");

// Per-sample device status (K2 RLE errors).
struct SampleStatus {
  int32_t kind;    // 0 ok, 1 "rle runs sum past n", 2 "rle runs sum to v, expected n"
  int32_t pad;
  int64_t value;
};

struct ScalarArgs {
  const int64_t* idx;        // count indices (device)
  int32_t count;
  int32_t n_fields;
  const uint64_t* cols[16];  // device columns, num_samples entries each
  uint64_t* outs[16];
};

struct LaunchArgs {
  const uint8_t* desc;       // count * desc_stride bytes (device)
  const uint8_t* payload;    // payload base (device): staged region or file image in HBM
  uint8_t* scratch;          // count * scratch_bytes (device)
  void* out;                 // count * out_sample_elems elements
  const void* lut;           // VAL_LUT: channels x 256 output values (exact, host-built)
  uint32_t* tables;          // K1 prologue tables: count x tab_stride u32
  SampleStatus* status;      // count entries
  int32_t count;
  ScalarArgs sc;             // column-walker K1: scalar fields gathered by the copy warp (n_fields 0: none)
  unsigned long long* ticket;  // column-walker K1: [0] next tile run, [1] CTAs done (self-resetting, zero between launches)
};

// One payload copy of a batch gathered by the device from the pinned, mapped host
// heap (zero-copy gather): `rows` rows of `row_bytes`, source rows `src_stride`
// apart from heap offset `src`, destination rows `dst_stride` (16-byte multiple)
// apart from slot offset `dst` (16-byte aligned).
struct GatherCopy {
  uint64_t src, dst;
  uint32_t row_bytes, rows, src_stride, dst_stride;
};
static_assert(sizeof(GatherCopy) == 32, "GatherCopy layout");

// kernels.cu
int launch_host_gather(const uint8_t* heap, uint64_t heap_bytes, uint8_t* slot, const GatherCopy* copies, int n,
                       void* stream);
int launch_rle_expand(const PlanDev& P, const LaunchArgs& A, void* stream);
int launch_image(const PlanDev& P, const LaunchArgs& A, void* stream);
int launch_array(const PlanDev& P, const LaunchArgs& A, void* stream);
int launch_scalar_gather(const ScalarArgs& S, void* stream);
int image_smem_bytes(const PlanDev& P);
SmemLayout img_layout_host(const PlanDev& P);
int image_tab_stride(const PlanDev& P);
int cw_smem_host(const PlanDev& P);

}  // namespace bbx
