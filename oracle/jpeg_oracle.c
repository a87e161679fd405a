/*
 * jpeg_oracle.c — CPU restatement of baseline JPEG decoding as the JPEG
 * codec extension of the bbox Decode transform (codec id 3).
 *
 * TEST INFRASTRUCTURE ONLY (see bbx_oracle.c's header): the checker for the
 * device decoder in paper_2306_12517_b200/csrc/jpeg.cu, never the product.
 *
 * The reference package has no JPEG codec (codecs.py:25-28 lists RAW, RLE,
 * SUBSAMPLE2), so there is no reference to pin against.  The
 * third-party decoder the FFCV north_star names is libjpeg-turbo (through
 * Pillow 12.2 in this image; `PIL.features.version("jpg")` = 6.2 API,
 * libjpeg-turbo 3.1.x).  This file restates the published algorithms that
 * library applies to a baseline, Huffman-coded, 8-bit, single-scan file with
 * its default decompression parameters (dct_method = JDCT_ISLOW,
 * do_fancy_upsampling = TRUE):
 *   - ITU-T T.81 Annex F.2.2 Huffman decoding, F.2.2.3 DECODE, F.2.2.1
 *     EXTEND; DC prediction reset at every RSTn (F.2.1.3.1); zero bits
 *     supplied once a marker is reached (libjpeg's fill_bit_buffer rule);
 *   - the "islow" integer IDCT (Loeffler-Ligtenberg-Moschytz, 13-bit
 *     constants, 2 extra bits between passes, output wrapped through a
 *     10-bit range-limit then clamped, IJG jidctint.c);
 *   - "fancy" triangle-filter chroma upsampling for h2v1 / h1v2 / h2v2 with
 *     edge replication (IJG jdsample.c; box replication when the downsampled
 *     width is <= 2);
 *   - JFIF YCbCr -> RGB with 16-bit fixed-point tables (IJG jdcolor.c).
 * Parity: pinned against Pillow's decoder on the fixtures committed under
 * tests/golden/ (tests/golden/make_jpeg_golden.py) — bit-exact, 0 LSB.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int code; char msg[256]; } or_err;   /* same layout as bbx_oracle.c */
enum { OJ_CORRUPT = 6 };

static const uint8_t kNatural[64 + 16] = {          /* zig-zag index -> natural index (T.81 Fig. A.6) */
  0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
  12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
  35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
  58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63,
  63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63, 63};  /* overrun guard */

typedef struct {
  int present;
  int32_t mincode[17], maxcode[18], valptr[17];
  uint8_t vals[256];
} oj_huff;

typedef struct {
  int id, h, v, tq, td, ta;
  int bw, bh;          /* coded blocks per row / column */
  int dw, dh;          /* downsampled_width / height */
  int16_t* coef;       /* bh*bw blocks of 64, natural order */
  uint8_t* plane;      /* (bh*8) x (bw*8) */
} oj_comp;

typedef struct {
  const uint8_t* d;
  int64_t n, pos;
  int bits, nbits;     /* bit buffer (msb first) */
  int marker;          /* a marker was reached: supply zeros */
} oj_reader;

static int fail(or_err* e, const char* m) {
  e->code = OJ_CORRUPT;
  snprintf(e->msg, sizeof e->msg, "jpeg: %s", m);
  return 1;
}

static int get_bit(oj_reader* r) {
  if (r->nbits == 0) {
    int b = 0;
    if (!r->marker && r->pos < r->n) {
      b = r->d[r->pos];
      if (b == 0xFF) {
        int b2 = r->pos + 1 < r->n ? r->d[r->pos + 1] : 0xD9;
        if (b2 == 0x00) r->pos += 2;
        else { r->marker = 1; b = 0; }
      } else {
        r->pos += 1;
      }
    }
    r->bits = b; r->nbits = 8;
  }
  r->nbits--;
  return (r->bits >> r->nbits) & 1;
}
static int receive(oj_reader* r, int s) {
  int v = 0;
  for (int i = 0; i < s; ++i) v = (v << 1) | get_bit(r);
  return v;
}
static int extend(int v, int s) { return s == 0 ? 0 : (v < (1 << (s - 1)) ? v - (1 << s) + 1 : v); }

static int huff_decode(oj_reader* r, const oj_huff* t, int* sym) {   /* T.81 F.16 */
  int code = get_bit(r), l = 1;
  while (l <= 16 && code > t->maxcode[l]) { code = (code << 1) | get_bit(r); ++l; }
  if (l > 16) return 1;
  *sym = t->vals[t->valptr[l] + code - t->mincode[l]];
  return 0;
}

static int build_huff(oj_huff* t, const uint8_t counts[16], const uint8_t* vals, int nvals, int is_dc) {
  int k = 0, code = 0;
  memset(t, 0, sizeof *t);
  if (is_dc)                                       /* DC symbols are categories 0..15 (jdhuff.c check) */
    for (int i = 0; i < nvals; ++i) if (vals[i] > 15) return 1;
  for (int l = 1; l <= 16; ++l) {
    t->valptr[l] = k;
    t->mincode[l] = code;
    code += counts[l - 1];
    k += counts[l - 1];
    t->maxcode[l] = counts[l - 1] ? code - 1 : -1;
    if (code >= (1 << l)) return 1;  /* over-subscribed, or an all-ones code */
    code <<= 1;
  }
  t->maxcode[17] = 0x7fffffff;
  if (k != nvals || k > 256) return 1;
  memcpy(t->vals, vals, (size_t)k);
  t->present = 1;
  return 0;
}

/* islow IDCT of one dequantized block (IJG jidctint.c algorithm) in 32-bit
 * arithmetic, as libjpeg-turbo's SIMD islow computes it (16-bit inputs,
 * 32-bit products and sums): identical to the C version's 64-bit JLONG for
 * every coefficient range a real 8-bit image produces (pinned on the Pillow
 * goldens); modular (wrapping) beyond, bit-identical to the device kernel. */
#define CB 13
#define P1 2
typedef uint32_t U32;
static int32_t desc32(U32 x, int n) { return (int32_t)(x + (1u << (n - 1))) >> n; }
static uint8_t range_out(int v) {                 /* range_limit[v & 1023] on the post-IDCT table */
  int s = ((v & 1023) ^ 512) - 512;
  s += 128;
  return (uint8_t)(s < 0 ? 0 : s > 255 ? 255 : s);
}
/* one 1-D pass over x[0..7] (stride st): outputs descaled by n bits */
static void idct_pass(const int32_t* x, int st, int32_t* o, int ost, int n) {
  U32 z1, z2, z3, z4, z5, t0, t1, t2, t3, t10, t11, t12, t13;
  z2 = (U32)x[2 * st]; z3 = (U32)x[6 * st];
  z1 = (z2 + z3) * 4433u;
  t2 = z1 + z3 * (U32)-15137;
  t3 = z1 + z2 * 6270u;
  t0 = ((U32)x[0] + (U32)x[4 * st]) << CB;
  t1 = ((U32)x[0] - (U32)x[4 * st]) << CB;
  t10 = t0 + t3; t13 = t0 - t3; t11 = t1 + t2; t12 = t1 - t2;
  t0 = (U32)x[7 * st]; t1 = (U32)x[5 * st]; t2 = (U32)x[3 * st]; t3 = (U32)x[st];
  z1 = t0 + t3; z2 = t1 + t2; z3 = t0 + t2; z4 = t1 + t3;
  z5 = (z3 + z4) * 9633u;
  t0 *= 2446u; t1 *= 16819u; t2 *= 25172u; t3 *= 12299u;
  z1 *= (U32)-7373; z2 *= (U32)-20995; z3 *= (U32)-16069; z4 *= (U32)-3196;
  z3 += z5; z4 += z5;
  t0 += z1 + z3; t1 += z2 + z4; t2 += z2 + z3; t3 += z1 + z4;
  o[0] = desc32(t10 + t3, n); o[7 * ost] = desc32(t10 - t3, n);
  o[ost] = desc32(t11 + t2, n); o[6 * ost] = desc32(t11 - t2, n);
  o[2 * ost] = desc32(t12 + t1, n); o[5 * ost] = desc32(t12 - t1, n);
  o[3 * ost] = desc32(t13 + t0, n); o[4 * ost] = desc32(t13 - t0, n);
}
static void idct_islow(const int16_t* coef, const uint16_t* q, uint8_t* out, int stride) {
  int32_t in[64], ws[64];
  for (int i = 0; i < 64; ++i) in[i] = (int32_t)((U32)(int32_t)coef[i] * (U32)q[i]);
  for (int c = 0; c < 8; ++c) {                   /* pass 1: columns (zero-AC shortcut is exact) */
    const int32_t* x = in + c;
    if (!x[8] && !x[16] && !x[24] && !x[32] && !x[40] && !x[48] && !x[56]) {
      for (int r = 0; r < 8; ++r) ws[r * 8 + c] = (int32_t)((U32)x[0] << P1);
      continue;
    }
    idct_pass(x, 8, ws + c, 8, CB - P1);
  }
  for (int r = 0; r < 8; ++r) {                   /* pass 2: rows */
    const int32_t* w = ws + r * 8;
    uint8_t* o = out + (size_t)r * stride;
    int32_t v[8];
    if (!w[1] && !w[2] && !w[3] && !w[4] && !w[5] && !w[6] && !w[7]) {
      const int32_t d = desc32((U32)w[0], P1 + 3);
      for (int c = 0; c < 8; ++c) v[c] = d;
    } else {
      idct_pass(w, 1, v, 1, CB + P1 + 3);
    }
    for (int c = 0; c < 8; ++c) o[c] = range_out(v[c]);
  }
}

/* Full-resolution sample (y, x) of component c, upsampled the libjpeg way. */
static int comp_sample(const oj_comp* c, int hmax, int vmax, int y, int x) {
  const int pw = c->bw * 8;
  const uint8_t* P = c->plane;
  const int rh = hmax / c->h, rv = vmax / c->v;
#define AT(yy, xx) ((int)P[(size_t)(yy) * pw + (xx)])
  if (rh == 1 && rv == 1) return AT(y, x);
  const int fancy_w = c->dw > 2;
  if (rh == 2 && rv == 1) {
    const int j = x >> 1;
    if (!fancy_w) return AT(y, j);
    const int jl = j > 0 ? j - 1 : 0, jr = j + 1 < c->dw ? j + 1 : c->dw - 1;
    return (x & 1) ? (3 * AT(y, j) + AT(y, jr) + 2) >> 2 : (3 * AT(y, j) + AT(y, jl) + 1) >> 2;
  }
  if (rh == 1 && rv == 2) {
    const int i = y >> 1;
    const int i1 = (y & 1) ? (i + 1 < c->dh ? i + 1 : c->dh - 1) : (i > 0 ? i - 1 : 0);
    return (3 * AT(i, x) + AT(i1, x) + ((y & 1) ? 2 : 1)) >> 2;
  }
  /* rh == 2 && rv == 2 */
  const int i = y >> 1, j = x >> 1;
  if (!fancy_w) return AT(i, j);
  const int i1 = (y & 1) ? (i + 1 < c->dh ? i + 1 : c->dh - 1) : (i > 0 ? i - 1 : 0);
  const int jn = (x & 1) ? (j + 1 < c->dw ? j + 1 : c->dw - 1) : (j > 0 ? j - 1 : 0);
  const int cs = 3 * AT(i, j) + AT(i1, j), ns = 3 * AT(i, jn) + AT(i1, jn);
  return (x & 1) ? (3 * cs + ns + 7) >> 4 : (3 * cs + ns + 8) >> 4;
#undef AT
}

static uint8_t clamp8(int v) { return (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v); }

#define FIX16(x) ((int)((x) * 65536.0 + 0.5))

int or_jpeg_decode(const uint8_t* d, int64_t n, int want_h, int want_w, int want_c, uint8_t* out, or_err* e) {
  oj_huff dc[4], ac[4];
  uint16_t qt[4][64];
  int qpresent[4] = {0};
  oj_comp comp[4];
  int ncomp = 0, height = 0, width = 0, restart = 0, sof = 0, rc = 1;
  int64_t scan = -1;
  memset(dc, 0, sizeof dc); memset(ac, 0, sizeof ac); memset(comp, 0, sizeof comp);
  char msg[160];
  if (n < 4 || d[0] != 0xFF || d[1] != 0xD8) return fail(e, "missing SOI marker");
  int64_t p = 2;
  while (scan < 0) {
    while (p < n && d[p] != 0xFF) ++p;                 /* garbage before a marker */
    while (p < n && d[p] == 0xFF) ++p;                 /* fill bytes */
    if (p + 2 >= n) return fail(e, "truncated header");
    int m = d[p++];
    if (m == 0xD8 || (m >= 0xD0 && m <= 0xD7) || m == 0x01) continue;
    if (m == 0xD9) return fail(e, "EOI before SOS");
    int len = (d[p] << 8) | d[p + 1];
    if (len < 2 || p + len > n) return fail(e, "truncated marker segment");
    const uint8_t* s = d + p + 2;
    int sl = len - 2;
    if (m == 0xC0 || m == 0xC1) {
      if (sof) return fail(e, "multiple SOF markers");
      sof = 1;
      if (sl < 6 || s[0] != 8) return fail(e, "unsupported sample precision");
      height = (s[1] << 8) | s[2]; width = (s[3] << 8) | s[4]; ncomp = s[5];
      if (ncomp != 1 && ncomp != 3) return fail(e, "unsupported component count");
      if (sl < 6 + 3 * ncomp) return fail(e, "truncated SOF");
      for (int i = 0; i < ncomp; ++i) {
        comp[i].id = s[6 + 3 * i];
        comp[i].h = s[7 + 3 * i] >> 4; comp[i].v = s[7 + 3 * i] & 15; comp[i].tq = s[8 + 3 * i];
        if (comp[i].h < 1 || comp[i].h > 2 || comp[i].v < 1 || comp[i].v > 2 || comp[i].tq > 3)
          return fail(e, "unsupported sampling factors");
      }
    } else if ((m >= 0xC2 && m <= 0xC3) || (m >= 0xC5 && m <= 0xC7) || (m >= 0xC9 && m <= 0xCB) ||
               (m >= 0xCD && m <= 0xCF)) {
      return fail(e, "unsupported JPEG process (progressive, lossless or arithmetic)");
    } else if (m == 0xC4) {
      int k = 0;
      while (k < sl) {
        if (k + 17 > sl) return fail(e, "truncated DHT");
        int tc = s[k] >> 4, th = s[k] & 15, tot = 0;
        for (int i = 0; i < 16; ++i) tot += s[k + 1 + i];
        if (tc > 1 || th > 3 || k + 17 + tot > sl) return fail(e, "bad DHT");
        if (build_huff(tc ? &ac[th] : &dc[th], s + k + 1, s + k + 17, tot, !tc)) return fail(e, "bad Huffman table");
        k += 17 + tot;
      }
    } else if (m == 0xDB) {
      int k = 0;
      while (k < sl) {
        int pq = s[k] >> 4, tq = s[k] & 15;
        if (tq > 3 || pq > 1 || k + 1 + 64 * (pq + 1) > sl) return fail(e, "bad DQT");
        for (int i = 0; i < 64; ++i)
          qt[tq][kNatural[i]] = pq ? (uint16_t)((s[k + 1 + 2 * i] << 8) | s[k + 2 + 2 * i]) : s[k + 1 + i];
        qpresent[tq] = 1;
        k += 1 + 64 * (pq + 1);
      }
    } else if (m == 0xDD) {
      if (sl < 2) return fail(e, "bad DRI");
      restart = (s[0] << 8) | s[1];
    } else if (m == 0xEE) {
      if (sl >= 12 && !memcmp(s, "Adobe", 5) && s[11] == 0 && ncomp == 3)
        return fail(e, "unsupported Adobe RGB (transform 0) JPEG");
    } else if (m == 0xDA) {
      if (!sof) return fail(e, "SOS before SOF");
      int ns = s[0];
      if (ns != ncomp || sl < 1 + 2 * ns + 3) return fail(e, "unsupported multi-scan JPEG");
      for (int i = 0; i < ns; ++i) {
        int cid = s[1 + 2 * i], j;
        for (j = 0; j < ncomp; ++j) if (comp[j].id == cid) break;
        if (j == ncomp || j != i) return fail(e, "SOS component order differs from SOF");
        comp[j].td = s[2 + 2 * i] >> 4; comp[j].ta = s[2 + 2 * i] & 15;
        if (comp[j].td > 3 || comp[j].ta > 3) return fail(e, "bad SOS table selector");
      }
      const uint8_t* t = s + 1 + 2 * ns;
      if (t[0] != 0 || t[1] != 63 || t[2] != 0) return fail(e, "not a baseline sequential scan");
      scan = p + len;
    }
    p += len;
  }
  if (height != want_h || width != want_w || ncomp != want_c) {
    snprintf(msg, sizeof msg, "header says %dx%dx%d, cell says %dx%dx%d", height, width, ncomp, want_h, want_w,
             want_c);
    return fail(e, msg);
  }
  if (height < 1 || width < 1) return fail(e, "empty image");
  int hmax = 1, vmax = 1;
  if (ncomp == 1) { comp[0].h = comp[0].v = 1; }
  for (int i = 0; i < ncomp; ++i) { if (comp[i].h > hmax) hmax = comp[i].h; if (comp[i].v > vmax) vmax = comp[i].v; }
  int mcus_x, mcus_y;
  if (ncomp == 1) {
    mcus_x = (width + 7) / 8; mcus_y = (height + 7) / 8;
  } else {
    mcus_x = (width + 8 * hmax - 1) / (8 * hmax); mcus_y = (height + 8 * vmax - 1) / (8 * vmax);
  }
  for (int i = 0; i < ncomp; ++i) {
    oj_comp* c = &comp[i];
    if (!qpresent[c->tq] || !dc[c->td].present || !ac[c->ta].present) return fail(e, "missing table");
    c->dw = (int)(((int64_t)width * c->h + hmax - 1) / hmax);
    c->dh = (int)(((int64_t)height * c->v + vmax - 1) / vmax);
    c->bw = ncomp == 1 ? mcus_x : mcus_x * c->h;
    c->bh = ncomp == 1 ? mcus_y : mcus_y * c->v;
    c->coef = calloc((size_t)c->bw * c->bh * 64, sizeof(int16_t));
    c->plane = malloc((size_t)c->bw * c->bh * 64);
    if (!c->coef || !c->plane) { fail(e, "out of memory"); goto done; }
  }
  {
    oj_reader r = {d, n, scan, 0, 0, 0};
    const int total = mcus_x * mcus_y;
    const int per = restart ? restart : total;
    int pred[4] = {0};
    for (int m = 0; m < total; ++m) {
      if (m && m % per == 0) {                      /* restart boundary: byte-align, expect RSTn */
        r.nbits = 0;
        int64_t q = r.pos;
        while (q + 1 < n && !(d[q] == 0xFF && d[q + 1] != 0 && d[q + 1] != 0xFF)) ++q;
        if (q + 1 >= n || d[q + 1] != 0xD0 + ((m / per - 1) & 7)) { fail(e, "missing restart marker"); goto done; }
        r.pos = q + 2; r.marker = 0;
        memset(pred, 0, sizeof pred);
      }
      const int mx = m % mcus_x, my = m / mcus_x;
      for (int ci = 0; ci < ncomp; ++ci) {
        oj_comp* c = &comp[ci];
        for (int v = 0; v < c->v; ++v)
          for (int h = 0; h < c->h; ++h) {
            int16_t* blk = c->coef + ((size_t)(my * c->v + v) * c->bw + (mx * c->h + h)) * 64;
            int t;
            if (huff_decode(&r, &dc[c->td], &t)) { fail(e, "bad Huffman code"); goto done; }
            int diff = t ? extend(receive(&r, t), t) : 0;
            pred[ci] += diff;
            blk[0] = (int16_t)pred[ci];
            for (int k = 1; k < 64; ++k) {
              int rs;
              if (huff_decode(&r, &ac[c->ta], &rs)) { fail(e, "bad Huffman code"); goto done; }
              int run = rs >> 4, sz = rs & 15;
              if (sz) {
                k += run;
                blk[kNatural[k]] = (int16_t)extend(receive(&r, sz), sz);
              } else if (run == 15) {
                k += 15;
              } else {
                break;
              }
            }
          }
      }
    }
  }
  for (int i = 0; i < ncomp; ++i) {
    oj_comp* c = &comp[i];
    for (int by = 0; by < c->bh; ++by)
      for (int bx = 0; bx < c->bw; ++bx)
        idct_islow(c->coef + ((size_t)by * c->bw + bx) * 64, qt[c->tq],
                   c->plane + (size_t)by * 8 * (c->bw * 8) + bx * 8, c->bw * 8);
  }
  {
    int crr[256], cbb[256], crg[256], cbg[256];
    for (int i = 0; i < 256; ++i) {
      int x = i - 128;
      crr[i] = (FIX16(1.40200) * x + 32768) >> 16;
      cbb[i] = (FIX16(1.77200) * x + 32768) >> 16;
      crg[i] = -FIX16(0.71414) * x;
      cbg[i] = -FIX16(0.34414) * x + 32768;
    }
    for (int y = 0; y < height; ++y)
      for (int x = 0; x < width; ++x) {
        uint8_t* o = out + ((size_t)y * width + x) * ncomp;
        if (ncomp == 1) { o[0] = (uint8_t)comp_sample(&comp[0], hmax, vmax, y, x); continue; }
        int Y = comp_sample(&comp[0], hmax, vmax, y, x);
        int cb = comp_sample(&comp[1], hmax, vmax, y, x);
        int cr = comp_sample(&comp[2], hmax, vmax, y, x);
        o[0] = clamp8(Y + crr[cr]);
        o[1] = clamp8(Y + ((cbg[cb] + crg[cr]) >> 16));
        o[2] = clamp8(Y + cbb[cb]);
      }
  }
  rc = 0;
done:
  for (int i = 0; i < 4; ++i) { free(comp[i].coef); free(comp[i].plane); }
  return rc;
}
