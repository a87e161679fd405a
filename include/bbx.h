/*
 * bbx.h — C ABI of the B200-native bbox loading hot path (libbbx.so).
 *
 * Plain C types only (no torch, no CUDA runtime types in signatures: CUDA
 * streams are passed as `void*` = cudaStream_t).  Every entry point replaces
 * one reference interface; the citations are to /root/reference/pkg/src/bbox.
 * The Python host mirror (paper_2306_12517_b200/) binds these with ctypes;
 * INTEGRATION.md shows the binding a maintainer of the reference would add.
 *
 * Error model: every call returns a bbx_status; the message of the last
 * failure on the calling thread is bbx_last_error().  Codes map 1:1 onto the
 * reference exception classes (errors.py:4-57).
 */
#ifndef BBX_H
#define BBX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BBX_OK = 0,
  BBX_INVALID_FILE = 1,        /* errors.InvalidFile */
  BBX_BAD_MAGIC = 2,           /* errors.BadMagic */
  BBX_UNSUPPORTED_VERSION = 3, /* errors.UnsupportedVersion */
  BBX_SCHEMA_MISMATCH = 4,     /* errors.SchemaMismatch */
  BBX_SPEC_MISMATCH = 5,       /* errors.SpecMismatch */
  BBX_CORRUPT_PAYLOAD = 6,     /* errors.CorruptPayload */
  BBX_INDEX_OUT_OF_RANGE = 7,  /* errors.IndexOutOfRange */
  BBX_CAPACITY_TOO_SMALL = 8,  /* errors.CapacityTooSmall */
  BBX_SHUTDOWN = 9,            /* errors.ShutdownError */
  BBX_CUDA_ERROR = 10,         /* device failure (no reference counterpart) */
  BBX_INVALID_HEADER = 11,     /* errors.InvalidHeader */
  BBX_INVALID_ARGUMENT = 12    /* ValueError */
} bbx_status;

/* Transform op kinds (pipeline.py:95-231 + extensions). */
typedef enum {
  BBX_OP_DECODE = 0,      /* Decode            pipeline.py:95-115  */
  BBX_OP_ARRAYREAD = 1,   /* ArrayRead         pipeline.py:118-129 */
  BBX_OP_TOFLOAT = 2,     /* ToFloat           pipeline.py:132-140 */
  BBX_OP_NORMALIZE = 3,   /* Normalize         pipeline.py:143-160 */
  BBX_OP_FLIP = 4,        /* RandomFlip        pipeline.py:163-181 */
  BBX_OP_CROP = 5,        /* RandomCrop        pipeline.py:184-202 */
  BBX_OP_RESIZE = 6,      /* Resize (nearest)  pipeline.py:205-231 */
  BBX_OP_RRC = 7,         /* extension: RandomResizedCrop decoder (bilinear) */
  BBX_OP_CENTERCROP = 8,  /* extension: CenterCrop decoder (bilinear) */
  BBX_OP_NORMALIZE_PC = 9,/* extension: per-channel NormalizeImage */
  BBX_OP_CAST = 10        /* extension: output cast f32 -> f16 / bf16 */
} bbx_op_kind;

typedef enum { BBX_U8 = 0, BBX_I64 = 1, BBX_F32 = 2, BBX_F64 = 3, BBX_F16 = 4, BBX_BF16 = 5 } bbx_dtype;

/* One compiled transform.  Same field meaning as the Transform constructor
 * arguments (RandomCrop(h, w), Resize(h, w), RandomFlip(p), Normalize(mean,
 * std)); RRC uses scale/ratio, CENTERCROP uses p as the crop ratio. */
typedef struct {
  int32_t kind;
  int32_t h, w;
  int32_t dtype;        /* BBX_OP_CAST target */
  double p;
  double scale[2];
  double ratio[2];
  float mean[4];
  float std[4];
} bbx_op;

typedef struct bbx_dataset bbx_dataset;
typedef struct bbx_loader bbx_loader;

/* Field description as decoded from the header (format.py:122-162). */
typedef struct {
  char name[64];
  int32_t kind;          /* FieldKind: 0 INT, 1 FLOAT, 2 FIXED_ARRAY, 3 VAR_BYTES, 4 IMAGE */
  int32_t array_dtype;   /* format.py:86-91 code: 0 u1, 1 i8, 2 f4, 3 f8 */
  int32_t ndims;
  int64_t dims[4];
  int32_t max_height, max_width, channels;
  int32_t cell_offset;   /* byte offset of the cell within a row */
} bbx_field_info;

typedef struct {
  int64_t num_samples;
  int64_t page_size;
  int64_t data_table_offset;
  int64_t heap_offset;
  int64_t alloc_table_offset;
  int32_t num_fields;
  int32_t row_width;
} bbx_header_info;

/* ---------------------------------------------------------------- dataset
 * Replaces reader.open_dataset / Dataset.__init__ (reader.py:323-366,
 * 535-546) for the OsCache strategy: mmap + decode_header (format.py:298-337). */
bbx_status bbx_dataset_open(const char* path, bbx_dataset** out);
void bbx_dataset_close(bbx_dataset* ds);                               /* reader.py:514-526 */
bbx_status bbx_dataset_header(const bbx_dataset* ds, bbx_header_info* out);
bbx_status bbx_dataset_field(const bbx_dataset* ds, int index, bbx_field_info* out);
/* Raw row bytes of sample i (reader.py:383-386 row_bytes). */
bbx_status bbx_dataset_row(const bbx_dataset* ds, int64_t i, uint8_t* out, int32_t out_len);
/* Device-resident heap: one-time upload of every heap page to HBM (the
 * B200 equivalent of ProcessCacheStrategy with capacity >= num_pages,
 * reader.py:67-77).  Batches then read payloads straight from HBM. */
bbx_status bbx_dataset_make_resident(bbx_dataset* ds, int device);
/* Pinned host copy of the heap (the OS-cache strategy's bytes held page-
 * locked): staged batches are then read by the copy engine with one batched
 * 2-D DMA call instead of a CPU gather.  threads <= 0: automatic. */
bbx_status bbx_dataset_pin_host(bbx_dataset* ds, int threads);
/* Page of sample i's first heap reference, -1 for all-inline (reader.py:430-437). */
bbx_status bbx_dataset_page_map(const bbx_dataset* ds, int64_t* out /* num_samples */);

/* ----------------------------------------------------------------- orders
 * TraversalOrder.epoch_indices (traversal.py:84-104): kind 0 sequential,
 * 1 random (rng.py:75-79 Fisher-Yates), 2 quasi-random (traversal.py:45-73).
 * page_map: per-sample page, -1 = None; may be NULL (all None).
 * Writes the permutation of 0..n-1 into out[n]. */
bbx_status bbx_epoch_order(int kind, uint64_t seed, uint64_t epoch, int64_t n, const int64_t* page_map,
                           int64_t batch_size, int64_t* out);

/* ----------------------------------------------------------------- loader
 * Replaces Loader.__init__ plan building (loader.py:153-198, PipelinePlan
 * pipeline.py:312-361) and the per-sample worker loop (loader.py:301-379,
 * 330-347) with one batch-granular device pipeline.
 *
 * staging_threads: host threads that gather payloads into pinned memory
 * (0 = automatic).  The loader owns pinned staging, device scratch, two
 * CUDA streams and per-slot events; outputs are caller-owned device buffers
 * bound per slot (bbx_loader_bind). */
bbx_status bbx_loader_create(bbx_dataset* ds, int device, int32_t batch_size, int32_t slot_count,
                             int32_t staging_threads, bbx_loader** out);
void bbx_loader_destroy(bbx_loader* ld);
/* Compile one field's chain (PipelinePlan, pipeline.py:312-361).  Opaque
 * stages are not expressible (BBX_SPEC_MISMATCH).  Returns the plan id and
 * the per-sample output spec (output_spec chain, pipeline.py:325-331). */
bbx_status bbx_loader_add_field(bbx_loader* ld, int32_t field_index, const bbx_op* ops, int32_t n_ops,
                                int32_t* plan_id, int64_t out_shape[4], int32_t* out_ndim, int32_t* out_dtype);
/* INT/FLOAT scalar column (loader.py:171-175, 188-193): gathered on device. */
bbx_status bbx_loader_add_scalar(bbx_loader* ld, int32_t field_index, int32_t* plan_id);
/* Bind slot `slot`'s output buffer for a plan: batch_size x out_shape elements. */
bbx_status bbx_loader_bind(bbx_loader* ld, int32_t plan_id, int32_t slot, void* out_dev);
/* Asynchronously produce one batch into `slot` (FillState + workers,
 * loader.py:301-379): indices idx[count] of the epoch order; per-sample
 * randomness from (seed, TAG_SAMPLE, epoch, index, field) (loader.py:339). */
bbx_status bbx_loader_submit(bbx_loader* ld, int32_t slot, const int64_t* idx, int32_t count, uint64_t seed,
                             uint64_t epoch);
/* Block until `slot` is filled (BatchRing.consume, pipeline.py:509-524).
 * On a per-sample failure returns its code, *bad_pos = lowest failing
 * position and bbx_last_error() = the reference's inner message.  The host
 * waits for the slot's device work only when the batch has device-detected
 * sample errors to read (RLE / JPEG fields) or is profiled; otherwise it
 * returns once the batch is queued, and bbx_loader_stream_wait orders the
 * consumer's stream after it. */
bbx_status bbx_loader_wait(bbx_loader* ld, int32_t slot, int64_t* bad_pos);
/* Make `stream` (a cudaStream_t) wait for slot's device work: no host block. */
bbx_status bbx_loader_stream_wait(bbx_loader* ld, int32_t slot, void* stream);
/* End of the consumer's lease on `slot` (BatchRing.end_consume,
 * pipeline.py:484-488): work queued on `stream` so far must finish before
 * the slot is overwritten.  stream may be NULL (legacy default stream). */
bbx_status bbx_loader_release(bbx_loader* ld, int32_t slot, void* stream);
/* One consumer step in one call (the Python iterator's per-batch sequence):
 * release_slot >= 0: bbx_loader_release(release_slot, stream); submit_slot >= 0:
 * bbx_loader_submit(submit_slot, idx, count, seed, epoch); then
 * bbx_loader_wait(wait_slot, bad_pos) and, when that succeeds,
 * bbx_loader_stream_wait(wait_slot, stream).  Returns the first failing
 * status (a wait failure carries bad_pos as bbx_loader_wait does). */
bbx_status bbx_loader_step(bbx_loader* ld, int32_t release_slot, int32_t submit_slot, const int64_t* idx,
                           int32_t count, uint64_t seed, uint64_t epoch, int32_t wait_slot, void* stream,
                           int64_t* bad_pos);
/* Wait for every submitted batch (used on shutdown / abandoned epochs). */
bbx_status bbx_loader_drain(bbx_loader* ld);

typedef struct {
  int64_t batches;
  int64_t samples;
  int64_t h2d_bytes;          /* host->device bytes copied */
  int64_t d2h_bytes;          /* device->host bytes copied (status words) */
  int64_t kernel_launches;    /* kernels launched by the loader */
  double stage_seconds;       /* host time spent gathering payloads */
  double wait_seconds;        /* consumer time blocked in bbx_loader_wait */
  /* profiling (bbx_loader_set_profiling): CUDA-event time of the per-field
   * transform kernels (K1 / array), measured on the loader's compute stream,
   * and their algorithmic bytes (source bytes the chain needs + output). */
  double kernel_seconds;
  int64_t kernel_timed;       /* kernel launches that were timed */
  int64_t kernel_bytes;       /* algorithmic bytes of the timed launches */
  int64_t zero_copy_bytes;    /* payload bytes kernels read straight from pinned host memory over PCIe */
  double  gap_seconds;        /* profiling: compute-stream idle between consecutive timed batches */
  double  h2d_late_seconds;   /* profiling: part of that idle time spent waiting for the batch's H2D */
  int64_t timed_batches;      /* profiling: batches whose kernel window (kernel_seconds) was timed */
  int64_t page_fetches;       /* page pool: pages fetched H2D (reader.py CacheStats.fetch_count) */
  int64_t page_reloads;       /* page pool: fetches of a page already fetched this epoch (reload_count) */
  int64_t io_reads;           /* Direct strategy: payload preads (reader.py io_read_count) */
  int64_t numa_node;          /* the GPU's NUMA node (-1: unknown); staging threads + pinned slots live there */
  int64_t staging_threads;    /* host gather threads */
  int64_t staging_cpus;       /* CPUs those threads are bound to (this rank's slice of the node; 0: unbound) */
  double  pipeline_seconds;   /* pipeline-thread time per batch: descriptors, staging, H2D and launch calls */
} bbx_loader_stats;
/* Zero-copy payloads: with a pinned host heap (bbx_dataset_pin_host) and no
 * RLE / JPEG fields, each sample's payload window comes straight from host
 * memory over PCIe -- no CPU gather, no staging copy: a gather kernel pulls the
 * batch's rows into the slot's HBM region (option "zc_gather", default), or K1
 * reads them itself ("zc_gather" 0).  Call before the first submit; ignored when
 * the plan cannot use it (RLE / JPEG plans stage their payloads). */
bbx_status bbx_loader_set_zero_copy(bbx_loader* ld, int enabled);
/* Loader tuning options (before the first submit; the defaults are the
 * measured-best settings):
 *   "window_staging"        1: stage only the rows x columns a RAW sample's chain reads
 *   "jpeg_header_cache"     1: keep each JPEG sample's parsed header for later epochs
 *   "jpeg_header_prefetch"  1: parse the headers of this loader's samples up front
 *   "jpeg_roi"              1: entropy-decode / IDCT only the MCUs the chain reads
 *   "parallel_desc_min"     256: batches of at least this many samples whose chains draw
 *                              RandomResizedCrop windows build their descriptors on the pool
 *   "cuda_graphs"           1: a full HBM-resident batch without per-sample device status
 *                              is captured once per (slot, compute stream) and replayed as a graph
 *   "direct_io"             0: Direct strategy -- every payload read is one pread of the whole
 *                              payload (reader.py:368-372), no window staging
 *   "read_latency_ns"       0: Direct: latency spun before each read (reader.py:369-370)
 *   "compute_streams"       2: consecutive batches alternate between two CUDA streams, so
 *                              one batch's kernels fill SMs the previous batch's tail leaves idle
 *   "zc_gather"             1: zero-copy payloads are gathered into HBM by a kernel before K1
 *                              (0: K1 reads the mapped host heap directly; fewer reads in flight)
 * Unknown names return BBX_INVALID_ARGUMENT. */
bbx_status bbx_loader_set_option(bbx_loader* ld, const char* name, int64_t value);
/* HBM page pool -- ProcessCacheStrategy (reader.py:152-297 ProcessCache,
 * loader.py:273-291,444-445): `capacity_pages` heap pages live in device memory.
 * Each epoch's plan (bbx_loader_plan_epoch, called before the epoch's first
 * submit, in epoch order) is the reference's PageSchedule: the trace of every
 * batch's samples' distinct pages, farthest-next-use eviction; a batch touching
 * more pages than the capacity fails with BBX_CAPACITY_TOO_SMALL ("batch
 * touches N pages, cache holds K").  Submitted batches then execute the plan
 * in order: each planned fetch copies one page H2D (mmap -> pinned -> pool
 * slot, `fetch_latency_s` spun first), and kernels read payloads from the pool.
 * Fetch / reload counts are the plan's (stats page_fetches / page_reloads).
 * Call set_page_pool before the first submit. */
bbx_status bbx_loader_set_page_pool(bbx_loader* ld, int64_t capacity_pages, double fetch_latency_s);
bbx_status bbx_loader_plan_epoch(bbx_loader* ld, const int64_t* idx, const int32_t* batch_len, int32_t n_batches,
                                 int64_t* planned_fetches, int64_t* planned_reloads);
/* Samples whose JPEG headers the loader parses up front (before the first
 * submit).  A distributed rank passes its shard of the first epoch so that
 * ranks do not each parse every header; others are parsed on first sight
 * and cached.  Without a call: every sample (single-process loaders). */
bbx_status bbx_loader_prefetch_headers(bbx_loader* ld, const int64_t* idx, int64_t n);
/* Turn per-launch CUDA-event timing of the transform kernels on/off. */
bbx_status bbx_loader_set_profiling(bbx_loader* ld, int enabled);   /* enabled > 1: every n-th batch */
bbx_status bbx_loader_get_stats(const bbx_loader* ld, bbx_loader_stats* out);
bbx_status bbx_loader_reset_stats(bbx_loader* ld);
/* The CUDA stream the loader's kernels run on (cudaStream_t as void*). */
void* bbx_loader_compute_stream(bbx_loader* ld);

/* ------------------------------------------------------------- one image
 * codecs.decode_image (codecs.py:91-128) on device: decode one blob into a
 * caller-owned (h, w, c) u8 device buffer.  Synchronous; for tests/tools.
 * codec: the cell's codec byte (format.py:72) -- BBX_CODEC_RAW / _RLE /
 * _SUBSAMPLE2 as codecs.py:25-28, plus BBX_CODEC_JPEG (this build's
 * extension: baseline JFIF, 1 or 3 components, sampling factors <= 2,
 * decoded bit-exactly as libjpeg-turbo's ISLOW + fancy-upsampling path). */
enum { BBX_CODEC_RAW = 0, BBX_CODEC_RLE = 1, BBX_CODEC_SUBSAMPLE2 = 2, BBX_CODEC_JPEG = 3 };
bbx_status bbx_decode_image(int32_t h, int32_t w, int32_t c, int32_t codec, const uint8_t* payload_host,
                            int64_t len, uint8_t* out_dev, int device);

/* The host half of the JPEG decode of one blob, without device work: header
 * (baseline sequential Huffman, 8-bit, 1 or 3 components, sampling <= 2),
 * dims == the cell's (h, w, c), Huffman tables, restart-marker count and
 * sequence.  BBX_OK or BBX_CORRUPT_PAYLOAD with the decoder's message.
 * validate_file (format.py:476-548, extended to codec 3) calls it per sample. */
bbx_status bbx_jpeg_check(int32_t h, int32_t w, int32_t c, const uint8_t* payload, int64_t len);

const char* bbx_last_error(void);
const char* bbx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BBX_H */
