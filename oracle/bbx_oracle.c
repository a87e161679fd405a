/*
 * bbx_oracle.c — CPU restatement of the reference `bbox` per-sample hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * `cpu_baseline` / `--impl reference` legs of bench.py may load this library,
 * and only as the checker / the timed CPU baseline.  The product path
 * (paper_2306_12517_b200/) never links or calls it.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function below
 * against golden vectors produced by the unmodified reference package
 * (tests/golden/make_golden.py): splitmix KATs, codec KATs + error texts, the
 * per-sample chain vectors, and whole-loader batches.  The extension ops
 * (random-resized-crop / center-crop bilinear decoders, per-channel
 * normalize, fp16/bf16 casts) have no reference counterpart; they are pinned
 * to OpenCV's INTER_LINEAR within +-1 LSB and to numpy's RN-even casts.
 *
 * Deliberately unfused and allocation-happy: every op writes a fresh buffer,
 * exactly like tests/oracles.py:reference_chain (oracles.py:181-199).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math: the
 * reference's Normalize is one IEEE f32 subtract and one IEEE f32 divide,
 * pipeline.py:158-160).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng ---
 * rng.py:23-79 — splitmix64 counter streams. */
#define GOLDEN 0x9E3779B97F4A7C15ULL

uint64_t or_mix64(uint64_t x) {                    /* rng.py:23-28 */
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
uint64_t or_fold(uint64_t s, uint64_t v) { return or_mix64(s + GOLDEN + v); } /* rng.py:31-33 */
uint64_t or_stream_seed(uint64_t seed, const uint64_t* parts, int n) {        /* rng.py:36-41 */
  uint64_t s = seed;
  for (int i = 0; i < n; ++i) s = or_fold(s, parts[i]);
  return s;
}
uint64_t or_next(uint64_t* st) { *st += GOLDEN; return or_mix64(*st); }      /* rng.py:57-59 */
uint64_t or_below(uint64_t* st, uint64_t n) { return or_next(st) % n; }      /* rng.py:61-65 */
int or_chance(uint64_t* st, double p) {                                      /* rng.py:67-73 */
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 1;
  uint64_t thr = (uint64_t)(p * 18446744073709551616.0); /* int(p * 2.0**64) */
  return or_next(st) < thr;
}
void or_shuffle(uint64_t* st, int64_t* a, int64_t n) {                      /* rng.py:75-79 */
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)or_below(st, (uint64_t)(i + 1));
    int64_t t = a[i]; a[i] = a[j]; a[j] = t;
  }
}
/* uniform double in [0,1) — extension draw for the RRC decoder (no reference). */
static double or_uniform(uint64_t* st) { return (double)(or_next(st) >> 11) * (1.0 / 9007199254740992.0); }

/* -------------------------------------------------------------- dtypes --- */
enum { DT_U8 = 0, DT_I64 = 1, DT_F32 = 2, DT_F64 = 3, DT_F16 = 4, DT_BF16 = 5 };
static int dt_size(int dt) {
  switch (dt) { case DT_U8: return 1; case DT_I64: return 8; case DT_F32: return 4;
                case DT_F64: return 8; default: return 2; }
}
static float load_f32(const void* p, int dt, int64_t i) {
  switch (dt) {
    case DT_U8: return (float)((const uint8_t*)p)[i];
    case DT_I64: return (float)((const int64_t*)p)[i];
    case DT_F32: return ((const float*)p)[i];
    case DT_F64: return (float)((const double*)p)[i];
  }
  return 0.f;
}
static uint16_t f32_to_bf16(float f) {           /* round-to-nearest-even */
  uint32_t u; memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static uint16_t f32_to_f16(float f) {
  _Float16 h = (_Float16)f; uint16_t u; memcpy(&u, &h, 2); return u;
}

/* ---------------------------------------------------------- errors -------
 * Mirrors errors.py class names; message texts follow codecs.py:91-128. */
enum { OR_OK = 0, OR_SCHEMA_MISMATCH = 4, OR_SPEC_MISMATCH = 5, OR_CORRUPT_PAYLOAD = 6 };
typedef struct { int code; char msg[256]; } or_err;

/* ----------------------------------------------------------- codecs ------
 * codecs.py:91-128.  Decodes into a dense (h, w, c) u8 buffer. */
enum { CODEC_RAW = 0, CODEC_RLE = 1, CODEC_SUB2 = 2, CODEC_JPEG = 3 };
/* jpeg_oracle.c: the JPEG codec extension (no reference counterpart). */
int or_jpeg_decode(const uint8_t* d, int64_t n, int h, int w, int c, uint8_t* out, or_err* e);

int or_decode_image(int h, int w, int c, int codec, const uint8_t* payload, int64_t len,
                    uint8_t* out, or_err* e) {
  int64_t n = (int64_t)h * w * c;
  if (codec == CODEC_RAW) {
    if (len != n) { e->code = OR_CORRUPT_PAYLOAD;
      snprintf(e->msg, sizeof e->msg, "raw payload is %lld bytes, expected %lld", (long long)len, (long long)n); return 1; }
    memcpy(out, payload, (size_t)n);
  } else if (codec == CODEC_RLE) {
    if (len % 5) { e->code = OR_CORRUPT_PAYLOAD;
      snprintf(e->msg, sizeof e->msg, "rle payload length is not a multiple of 5"); return 1; }
    int64_t pos = 0;
    for (int64_t off = 0; off < len; off += 5) {
      uint32_t cnt = (uint32_t)payload[off] | (uint32_t)payload[off + 1] << 8 |
                     (uint32_t)payload[off + 2] << 16 | (uint32_t)payload[off + 3] << 24;
      uint8_t v = payload[off + 4];
      if (cnt == 0 || pos + (int64_t)cnt > n) { e->code = OR_CORRUPT_PAYLOAD;
        snprintf(e->msg, sizeof e->msg, "rle runs sum past %lld bytes", (long long)n); return 1; }
      memset(out + pos, v, cnt);
      pos += cnt;
    }
    if (pos != n) { e->code = OR_CORRUPT_PAYLOAD;
      snprintf(e->msg, sizeof e->msg, "rle runs sum to %lld bytes, expected %lld", (long long)pos, (long long)n); return 1; }
  } else if (codec == CODEC_SUB2) {
    int sh = (h + 1) / 2, sw = (w + 1) / 2;
    if (len != (int64_t)sh * sw * c) { e->code = OR_CORRUPT_PAYLOAD;
      snprintf(e->msg, sizeof e->msg, "subsampled payload is %lld bytes, expected %lld", (long long)len,
               (long long)sh * sw * c); return 1; }
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        for (int k = 0; k < c; ++k)
          out[((int64_t)y * w + x) * c + k] = payload[((int64_t)(y / 2) * sw + x / 2) * c + k];
  } else if (codec == CODEC_JPEG) {
    return or_jpeg_decode(payload, len, h, w, c, out, e);
  } else {
    e->code = OR_CORRUPT_PAYLOAD; snprintf(e->msg, sizeof e->msg, "unknown codec %d", codec); return 1;
  }
  return 0;
}

/* --------------------------------------------------------------- ops -----
 * pipeline.py:95-231 plus the extension decoders. */
enum {
  OP_DECODE = 0, OP_ARRAYREAD = 1, OP_TOFLOAT = 2, OP_NORMALIZE = 3, OP_FLIP = 4, OP_CROP = 5,
  OP_RESIZE = 6, OP_RRC = 7, OP_CENTERCROP = 8, OP_NORMALIZE_PC = 9, OP_CAST = 10
};
typedef struct {
  int32_t kind;
  int32_t h, w;        /* crop / resize / decoder output size */
  int32_t dtype;       /* OP_CAST target */
  double p;            /* flip probability; center-crop ratio */
  double scale[2];     /* RRC */
  double ratio[2];     /* RRC */
  float mean[4], std[4]; /* OP_NORMALIZE uses [0]; OP_NORMALIZE_PC uses [0..c) */
} or_op;

typedef struct { void* data; int ndim; int64_t shape[4]; int dtype; } or_buf;

static int64_t nelem(const or_buf* b) { int64_t n = 1; for (int i = 0; i < b->ndim; ++i) n *= b->shape[i]; return n; }
static void buf_alloc(or_buf* b) { b->data = calloc((size_t)(nelem(b) > 0 ? nelem(b) : 1), (size_t)dt_size(b->dtype)); }

/* Bilinear resample of a (ch x cw) window at (top, left) of an (h, w, c) u8
 * image to (oh, ow, c).  Extension (no reference): half-pixel centres and
 * replicated borders like OpenCV INTER_LINEAR, with 11-bit integer weights so
 * the CPU and the GPU agree bit for bit. */
static void lin_axis(int o, int out_n, int in_n, int* i0, int* i1, int* w1) {
  int64_t num = (int64_t)(2 * o + 1) * in_n - out_n, den = 2 * (int64_t)out_n;
  if (num <= 0) { *i0 = 0; *i1 = 0; *w1 = 0; return; }
  int64_t q = num / den, r = num % den;
  if (q >= in_n - 1) { *i0 = in_n - 1; *i1 = in_n - 1; *w1 = 0; return; }
  *i0 = (int)q; *i1 = (int)q + 1; *w1 = (int)((r * 2048 + den / 2) / den);
}
static void resample_bilinear(const uint8_t* img, int w, int c, int top, int left, int ch, int cw,
                              uint8_t* out, int oh, int ow) {
  for (int y = 0; y < oh; ++y) {
    int y0, y1, wy; lin_axis(y, oh, ch, &y0, &y1, &wy);
    for (int x = 0; x < ow; ++x) {
      int x0, x1, wx; lin_axis(x, ow, cw, &x0, &x1, &wx);
      const uint8_t* r0 = img + ((int64_t)(top + y0) * w + left) * c;
      const uint8_t* r1 = img + ((int64_t)(top + y1) * w + left) * c;
      for (int k = 0; k < c; ++k) {
        uint32_t a = (uint32_t)(2048 - wx) * r0[x0 * c + k] + (uint32_t)wx * r0[x1 * c + k];
        uint32_t b = (uint32_t)(2048 - wx) * r1[x0 * c + k] + (uint32_t)wx * r1[x1 * c + k];
        out[((int64_t)y * ow + x) * c + k] = (uint8_t)(((uint32_t)(2048 - wy) * a + (uint32_t)wy * b + (1u << 21)) >> 22);
      }
    }
  }
}

/* RandomResizedCrop window (extension; torchvision/FFCV get_params rule with
 * bbox Rng draws).  Returns top, left, ch, cw within an h x w image. */
void or_rrc_window(uint64_t* st, int h, int w, const double scale[2], const double ratio[2],
                   int* top, int* left, int* ch, int* cw) {
  double area = (double)h * (double)w;
  double lr0 = log(ratio[0]), lr1 = log(ratio[1]);
  for (int attempt = 0; attempt < 10; ++attempt) {
    double target = area * (scale[0] + (scale[1] - scale[0]) * or_uniform(st));
    double aspect = exp(lr0 + (lr1 - lr0) * or_uniform(st));
    int ww = (int)nearbyint(sqrt(target * aspect));
    int hh = (int)nearbyint(sqrt(target / aspect));
    if (ww > 0 && ww <= w && hh > 0 && hh <= h) {
      *top = (int)or_below(st, (uint64_t)(h - hh + 1));
      *left = (int)or_below(st, (uint64_t)(w - ww + 1));
      *ch = hh; *cw = ww; return;
    }
  }
  double in_ratio = (double)w / (double)h;
  int ww, hh;
  if (in_ratio < ratio[0]) { ww = w; hh = (int)nearbyint(ww / ratio[0]); }
  else if (in_ratio > ratio[1]) { hh = h; ww = (int)nearbyint(hh * ratio[1]); }
  else { ww = w; hh = h; }
  if (hh < 1) hh = 1;
  if (ww < 1) ww = 1;
  if (hh > h) hh = h;
  if (ww > w) ww = w;
  *top = (h - hh) / 2; *left = (w - ww) / 2; *ch = hh; *cw = ww;
}
/* CenterCrop window (extension; FFCV get_center_crop: side = int(ratio*min(h,w))). */
void or_center_window(int h, int w, double ratio, int* top, int* left, int* ch, int* cw) {
  int s = h < w ? h : w;
  int c = (int)(ratio * (double)s);
  if (c < 1) c = 1;
  *top = (h - c) / 2; *left = (w - c) / 2; *ch = c; *cw = c;
}

/* One sample through a chain.  src: image → (cell dims + payload);
 * array → payload bytes of an (adims, adtype) array. */
typedef struct {
  int is_image;
  int max_h, max_w, channels;       /* image field descriptor */
  int h, w, c, codec;               /* image cell */
  int andim; int64_t adims[4]; int adtype; /* array field */
  const uint8_t* payload; int64_t len;
} or_source;

int or_run_chain(const or_op* ops, int n_ops, const or_source* src, uint64_t rng_state,
                 or_buf* result, uint64_t* state_out, or_err* e) {
  uint64_t st = rng_state;
  or_buf cur = {0};
  e->code = 0; e->msg[0] = 0;
  for (int oi = 0; oi < n_ops; ++oi) {
    const or_op* op = &ops[oi];
    or_buf nb = {0};
    if (oi == 0) {
      if (op->kind == OP_DECODE) {                     /* pipeline.py:106-115 */
        nb.ndim = 3; nb.shape[0] = src->max_h; nb.shape[1] = src->max_w; nb.shape[2] = src->channels;
        nb.dtype = DT_U8; buf_alloc(&nb);
        int vh = src->h < src->max_h ? src->h : src->max_h, vw = src->w < src->max_w ? src->w : src->max_w;
        if (src->h > src->max_h || src->w > src->max_w || src->c != src->channels) {
          e->code = OR_SCHEMA_MISMATCH;
          snprintf(e->msg, sizeof e->msg, "output buffer must be u8 (%d, %d, %d), got uint8 (%d, %d, %d)",
                   src->h, src->w, src->c, vh, vw, src->channels);
          free(nb.data); return 1;
        }
        uint8_t* tmp = malloc((size_t)src->h * src->w * src->c + 1);
        if (or_decode_image(src->h, src->w, src->c, src->codec, src->payload, src->len, tmp, e)) {
          free(tmp); free(nb.data); return 1;
        }
        for (int y = 0; y < src->h; ++y)
          memcpy((uint8_t*)nb.data + (int64_t)y * src->max_w * src->c, tmp + (int64_t)y * src->w * src->c,
                 (size_t)src->w * src->c);
        free(tmp);
      } else if (op->kind == OP_RRC || op->kind == OP_CENTERCROP) {   /* extension decoders */
        if (src->h > src->max_h || src->w > src->max_w || src->c != src->channels) {
          e->code = OR_SCHEMA_MISMATCH;
          snprintf(e->msg, sizeof e->msg, "image %dx%dx%d does not fit field (%d, %d, %d)", src->h, src->w,
                   src->c, src->max_h, src->max_w, src->channels);
          return 1;
        }
        uint8_t* tmp = malloc((size_t)src->h * src->w * src->c + 1);
        if (or_decode_image(src->h, src->w, src->c, src->codec, src->payload, src->len, tmp, e)) {
          free(tmp); return 1;
        }
        int top, left, ch, cw;
        if (op->kind == OP_RRC) or_rrc_window(&st, src->h, src->w, op->scale, op->ratio, &top, &left, &ch, &cw);
        else or_center_window(src->h, src->w, op->p, &top, &left, &ch, &cw);
        nb.ndim = 3; nb.shape[0] = op->h; nb.shape[1] = op->w; nb.shape[2] = src->c; nb.dtype = DT_U8;
        buf_alloc(&nb);
        resample_bilinear(tmp, src->w, src->c, top, left, ch, cw, (uint8_t*)nb.data, op->h, op->w);
        free(tmp);
      } else if (op->kind == OP_ARRAYREAD) {           /* pipeline.py:128-129 */
        nb.ndim = src->andim; memcpy(nb.shape, src->adims, sizeof nb.shape); nb.dtype = src->adtype;
        buf_alloc(&nb);
        memcpy(nb.data, src->payload, (size_t)src->len);
      } else {
        e->code = OR_SPEC_MISMATCH; snprintf(e->msg, sizeof e->msg, "first op must be a source"); return 1;
      }
    } else {
      int64_t n = nelem(&cur);
      int isz = dt_size(cur.dtype);
      switch (op->kind) {
        case OP_TOFLOAT:                               /* pipeline.py:139-140 */
          nb = cur; nb.dtype = DT_F32; buf_alloc(&nb);
          for (int64_t i = 0; i < n; ++i) ((float*)nb.data)[i] = load_f32(cur.data, cur.dtype, i);
          break;
        case OP_NORMALIZE: {                           /* pipeline.py:158-160 */
          nb = cur; nb.dtype = DT_F32; buf_alloc(&nb);
          float m = op->mean[0], s = op->std[0];
          for (int64_t i = 0; i < n; ++i) {
            float v = load_f32(cur.data, cur.dtype, i) - m;
            ((float*)nb.data)[i] = v / s;
          }
          break;
        }
        case OP_NORMALIZE_PC: {                        /* extension: per-channel */
          nb = cur; nb.dtype = DT_F32; buf_alloc(&nb);
          int64_t c = cur.shape[cur.ndim - 1];
          for (int64_t i = 0; i < n; ++i) {
            int k = (int)(i % c);
            float v = load_f32(cur.data, cur.dtype, i) - op->mean[k];
            ((float*)nb.data)[i] = v / op->std[k];
          }
          break;
        }
        case OP_CAST: {                                /* extension: f32 -> f16/bf16/f32 */
          nb = cur; nb.dtype = op->dtype; buf_alloc(&nb);
          for (int64_t i = 0; i < n; ++i) {
            float v = load_f32(cur.data, cur.dtype, i);
            if (op->dtype == DT_F16) ((uint16_t*)nb.data)[i] = f32_to_f16(v);
            else if (op->dtype == DT_BF16) ((uint16_t*)nb.data)[i] = f32_to_bf16(v);
            else ((float*)nb.data)[i] = v;
          }
          break;
        }
        case OP_FLIP: {                                /* pipeline.py:177-181 */
          nb = cur; buf_alloc(&nb);
          int flip = or_chance(&st, op->p);
          int64_t H = cur.shape[0], W = cur.shape[1], C = cur.shape[2];
          for (int64_t y = 0; y < H; ++y)
            for (int64_t x = 0; x < W; ++x) {
              int64_t sx = flip ? W - 1 - x : x;
              memcpy((uint8_t*)nb.data + ((y * W + x) * C) * isz, (uint8_t*)cur.data + ((y * W + sx) * C) * isz,
                     (size_t)(C * isz));
            }
          break;
        }
        case OP_CROP: {                                /* pipeline.py:199-202 */
          int64_t H = cur.shape[0], W = cur.shape[1], C = cur.shape[2];
          int64_t top = (int64_t)or_below(&st, (uint64_t)(H - op->h + 1));
          int64_t left = (int64_t)or_below(&st, (uint64_t)(W - op->w + 1));
          nb = cur; nb.shape[0] = op->h; nb.shape[1] = op->w; buf_alloc(&nb);
          for (int64_t y = 0; y < op->h; ++y)
            memcpy((uint8_t*)nb.data + (y * op->w * C) * isz, (uint8_t*)cur.data + (((top + y) * W + left) * C) * isz,
                   (size_t)(op->w * C * isz));
          break;
        }
        case OP_RESIZE: {                              /* pipeline.py:221-231 */
          int64_t H = cur.shape[0], W = cur.shape[1], C = cur.shape[2];
          nb = cur; nb.shape[0] = op->h; nb.shape[1] = op->w; buf_alloc(&nb);
          for (int64_t y = 0; y < op->h; ++y)
            for (int64_t x = 0; x < op->w; ++x) {
              int64_t sy = y * H / op->h, sx = x * W / op->w;
              memcpy((uint8_t*)nb.data + ((y * op->w + x) * C) * isz, (uint8_t*)cur.data + ((sy * W + sx) * C) * isz,
                     (size_t)(C * isz));
            }
          break;
        }
        default:
          e->code = OR_SPEC_MISMATCH; snprintf(e->msg, sizeof e->msg, "unsupported op %d", op->kind);
          free(cur.data); return 1;
      }
    }
    free(cur.data);
    cur = nb;
  }
  *result = cur;
  if (state_out) *state_out = st;
  return 0;
}

/* ------------------------------------------------------- batch runner -----
 * The per-batch CPU baseline: the work loader.py:_process_position
 * (loader.py:330-347) does for one field, for `count` samples, on
 * `nthreads` pthreads.  Rows come from the mmap'd data table; payloads are
 * views into the mmap'd heap (reader.py:439-466, OsCache).  Output is the
 * batch tensor (count, *out_shape) in out_dtype. */
typedef struct {
  const uint8_t* file; const uint8_t* rows; int64_t row_width; int64_t cell_off;
  int is_image; int max_h, max_w, channels; int andim; int64_t adims[4]; int adtype; int64_t anbytes;
  const or_op* ops; int n_ops;
  const int64_t* idx; int64_t count; uint64_t seed, epoch, fidx;
  uint8_t* out; int64_t out_sample_bytes;
  int64_t next; pthread_mutex_t mu;
  int64_t bad_pos; or_err err;
} or_batch;

static void* batch_worker(void* arg) {
  or_batch* b = arg;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    int64_t pos = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (pos >= b->count) break;
    int64_t i = b->idx[pos];
    const uint8_t* cell = b->rows + i * b->row_width + b->cell_off;
    or_source s; memset(&s, 0, sizeof s);
    s.is_image = b->is_image;
    if (b->is_image) {                                 /* format.py:72 <QQHHBB2x> */
      uint64_t off, len; uint16_t h, w;
      memcpy(&off, cell, 8); memcpy(&len, cell + 8, 8); memcpy(&h, cell + 16, 2); memcpy(&w, cell + 18, 2);
      s.h = h; s.w = w; s.c = cell[20]; s.codec = cell[21];
      s.max_h = b->max_h; s.max_w = b->max_w; s.channels = b->channels;
      s.payload = b->file + off; s.len = (int64_t)len;
    } else {
      uint64_t off; memcpy(&off, cell, 8);
      s.andim = b->andim; memcpy(s.adims, b->adims, sizeof s.adims); s.adtype = b->adtype;
      s.payload = b->file + off; s.len = b->anbytes;
    }
    uint64_t parts[4] = {2, b->epoch, (uint64_t)i, b->fidx};  /* loader.py:339, TAG_SAMPLE=2 */
    uint64_t st = or_stream_seed(b->seed, parts, 4);
    or_buf r; or_err e;
    if (or_run_chain(b->ops, b->n_ops, &s, st, &r, NULL, &e)) {
      pthread_mutex_lock(&b->mu);
      if (b->bad_pos < 0 || pos < b->bad_pos) { b->bad_pos = pos; b->err = e; }
      pthread_mutex_unlock(&b->mu);
      continue;
    }
    memcpy(b->out + pos * b->out_sample_bytes, r.data, (size_t)b->out_sample_bytes);
    free(r.data);
  }
  return NULL;
}

/* Returns 0 on success; on a per-sample failure returns the error code and
 * fills *bad_pos / msg (the lowest failing position, loader.py:400-402). */
int or_run_batch(const uint8_t* file, const uint8_t* rows, int64_t row_width, int64_t cell_off,
                 int is_image, int max_h, int max_w, int channels,
                 int andim, const int64_t* adims, int adtype, int64_t anbytes,
                 const or_op* ops, int n_ops, const int64_t* idx, int64_t count,
                 uint64_t seed, uint64_t epoch, uint64_t fidx,
                 uint8_t* out, int64_t out_sample_bytes, int nthreads,
                 int64_t* bad_pos, char* msg, int msg_len) {
  or_batch b; memset(&b, 0, sizeof b);
  b.file = file; b.rows = rows; b.row_width = row_width; b.cell_off = cell_off;
  b.is_image = is_image; b.max_h = max_h; b.max_w = max_w; b.channels = channels;
  b.andim = andim; for (int k = 0; k < 4 && k < andim; ++k) b.adims[k] = adims[k];
  b.adtype = adtype; b.anbytes = anbytes;
  b.ops = ops; b.n_ops = n_ops; b.idx = idx; b.count = count; b.seed = seed; b.epoch = epoch; b.fidx = fidx;
  b.out = out; b.out_sample_bytes = out_sample_bytes; b.bad_pos = -1;
  pthread_mutex_init(&b.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) batch_worker(&b);
  else {
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &b);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&b.mu);
  *bad_pos = b.bad_pos;
  if (b.bad_pos >= 0) {
    snprintf(msg, (size_t)msg_len, "%s", b.err.msg);
    return b.err.code;
  }
  return 0;
}

/* Single-sample entry for the chain-vector tests. */
int or_chain_one(const or_op* ops, int n_ops, int is_image, int max_h, int max_w, int channels,
                 int h, int w, int c, int codec, int andim, const int64_t* adims, int adtype,
                 const uint8_t* payload, int64_t len, uint64_t rng_state,
                 uint8_t* out, int64_t out_cap, int64_t* out_shape, int* out_ndim, int* out_dtype,
                 uint64_t* state_out, char* msg, int msg_len) {
  or_source s; memset(&s, 0, sizeof s);
  s.is_image = is_image; s.max_h = max_h; s.max_w = max_w; s.channels = channels;
  s.h = h; s.w = w; s.c = c; s.codec = codec; s.andim = andim; s.adtype = adtype;
  for (int k = 0; k < andim && k < 4; ++k) s.adims[k] = adims[k];
  s.payload = payload; s.len = len;
  or_buf r; or_err e;
  if (or_run_chain(ops, n_ops, &s, rng_state, &r, state_out, &e)) {
    snprintf(msg, (size_t)msg_len, "%s", e.msg);
    return e.code;
  }
  int64_t nb = nelem(&r) * dt_size(r.dtype);
  if (nb > out_cap) { free(r.data); snprintf(msg, (size_t)msg_len, "out buffer too small"); return OR_SPEC_MISMATCH; }
  memcpy(out, r.data, (size_t)nb);
  *out_ndim = r.ndim; for (int k = 0; k < r.ndim; ++k) out_shape[k] = r.shape[k];
  *out_dtype = r.dtype;
  free(r.data);
  return 0;
}
