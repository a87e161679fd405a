// JPEG header parsing and Huffman table construction (host side of codec 3).
//
// The reference has no JPEG codec (codecs.py:25-28); this is the extension
// BASELINE.json's north_star asks for.  Accepted: baseline / extended
// sequential Huffman (SOF0/SOF1), 8-bit, 1 or 3 components, sampling factors
// in {1, 2}, one interleaved scan (Ss=0, Se=63, Ah=Al=0), optional DRI.
// Everything else is rejected with a CorruptPayload reason (no fallback).
#include <cstdio>
#include <cstring>

#include "jpeg.h"

namespace bbx {

static const uint8_t kZigzagToNatural[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
    41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
    30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

int jpeg_parse_header(const uint8_t* d, uint64_t n, JpegHeader* h, char* err, int errlen) {
  auto bad = [&](const char* m) { std::snprintf(err, errlen, "jpeg: %s", m); return 1; };
  if (n < 4 || d[0] != 0xFF || d[1] != 0xD8) return bad("missing SOI marker");
  uint64_t p = 2;
  bool sof = false;
  for (;;) {
    while (p < n && d[p] != 0xFF) ++p;
    while (p < n && d[p] == 0xFF) ++p;
    if (p + 2 >= n) return bad("truncated header");
    const int m = d[p++];
    if (m == 0xD8 || (m >= 0xD0 && m <= 0xD7) || m == 0x01) continue;
    if (m == 0xD9) return bad("EOI before SOS");
    const int len = (d[p] << 8) | d[p + 1];
    if (len < 2 || p + len > n) return bad("truncated marker segment");
    const uint8_t* s = d + p + 2;
    const int sl = len - 2;
    if (m == 0xC0 || m == 0xC1) {
      if (sof) return bad("multiple SOF markers");
      sof = true;
      if (sl < 6 || s[0] != 8) return bad("unsupported sample precision");
      h->height = (s[1] << 8) | s[2];
      h->width = (s[3] << 8) | s[4];
      h->ncomp = s[5];
      if (h->ncomp != 1 && h->ncomp != 3) return bad("unsupported component count");
      if (sl < 6 + 3 * h->ncomp) return bad("truncated SOF");
      for (int i = 0; i < h->ncomp; ++i) {
        auto& c = h->comp[i];
        c.id = s[6 + 3 * i];
        c.h = s[7 + 3 * i] >> 4;
        c.v = s[7 + 3 * i] & 15;
        c.tq = s[8 + 3 * i];
        c.td = c.ta = 0;
        if (c.h < 1 || c.h > 2 || c.v < 1 || c.v > 2 || c.tq > 3) return bad("unsupported sampling factors");
      }
    } else if ((m >= 0xC2 && m <= 0xC3) || (m >= 0xC5 && m <= 0xC7) || (m >= 0xC9 && m <= 0xCB) ||
               (m >= 0xCD && m <= 0xCF)) {
      return bad("unsupported JPEG process (progressive, lossless or arithmetic)");
    } else if (m == 0xC4) {
      int k = 0;
      while (k < sl) {
        if (k + 17 > sl) return bad("truncated DHT");
        const int tc = s[k] >> 4, th = s[k] & 15;
        int tot = 0;
        for (int i = 0; i < 16; ++i) tot += s[k + 1 + i];
        if (tc > 1 || th > 3 || tot > 256 || k + 17 + tot > sl) return bad("bad DHT");
        JpegHeader::Huff& t = tc ? h->ac[th] : h->dc[th];
        t.present = true;
        std::memcpy(t.counts, s + k + 1, 16);
        std::memcpy(t.vals, s + k + 17, tot);
        t.nvals = tot;
        k += 17 + tot;
      }
    } else if (m == 0xDB) {
      int k = 0;
      while (k < sl) {
        const int pq = s[k] >> 4, tq = s[k] & 15;
        if (tq > 3 || pq > 1 || k + 1 + 64 * (pq + 1) > sl) return bad("bad DQT");
        for (int i = 0; i < 64; ++i)
          h->qt[tq].q[kZigzagToNatural[i]] =
              pq ? (uint16_t)((s[k + 1 + 2 * i] << 8) | s[k + 2 + 2 * i]) : (uint16_t)s[k + 1 + i];
        h->qt[tq].present = true;
        k += 1 + 64 * (pq + 1);
      }
    } else if (m == 0xDD) {
      if (sl < 2) return bad("bad DRI");
      h->restart = (s[0] << 8) | s[1];
    } else if (m == 0xEE) {
      if (sl >= 12 && !std::memcmp(s, "Adobe", 5) && s[11] == 0 && h->ncomp == 3)
        return bad("unsupported Adobe RGB (transform 0) JPEG");
    } else if (m == 0xDA) {
      if (!sof) return bad("SOS before SOF");
      const int ns = s[0];
      if (ns != h->ncomp || sl < 1 + 2 * ns + 3) return bad("unsupported multi-scan JPEG");
      for (int i = 0; i < ns; ++i) {
        if (s[1 + 2 * i] != h->comp[i].id) return bad("SOS component order differs from SOF");
        h->comp[i].td = s[2 + 2 * i] >> 4;
        h->comp[i].ta = s[2 + 2 * i] & 15;
        if (h->comp[i].td > 3 || h->comp[i].ta > 3) return bad("bad SOS table selector");
      }
      const uint8_t* t = s + 1 + 2 * ns;
      if (t[0] != 0 || t[1] != 63 || t[2] != 0) return bad("not a baseline sequential scan");
      h->scan_off = (uint32_t)(p + len);
      break;
    }
    p += len;
  }
  if (h->width < 1 || h->height < 1) return bad("empty image");
  if (h->ncomp == 1) h->comp[0].h = h->comp[0].v = 1;
  for (int i = 0; i < h->ncomp; ++i) {
    const auto& c = h->comp[i];
    if (!h->qt[c.tq].present || !h->dc[c.td].present || !h->ac[c.ta].present) return bad("missing table");
  }
  return 0;
}

// Canonical code assignment (T.81 C.2, F.15): per length, codes are
// consecutive.  The fast table resolves every code of <= kJpegFastBits bits
// to (length, extra bits, zero run, end of block).
bool jpeg_build_huff(const JpegHeader::Huff& t, bool is_ac, JHuff* o) {
  std::memset(o, 0, sizeof *o);
  if (!is_ac)
    for (int i = 0; i < t.nvals; ++i) if (t.vals[i] > 15) return false;   // DC categories (jdhuff.c check)
  constexpr int F = kJpegFastBits;
  int k = 0, code = 0;
  for (int l = 1; l <= 16; ++l) {
    const int cnt = t.counts[l - 1];
    o->valoff[l] = k - code;
    o->maxcode[l] = cnt ? code + cnt - 1 : -1;
    for (int i = 0; i < cnt; ++i, ++k, ++code) {
      if (code >= (1 << l) || k >= 256) return false;
      if (l > F) continue;
      const int sym = t.vals[k];
      const int size = is_ac ? (sym & 15) : sym, run = is_ac ? (sym >> 4) : 0;
      const int sh = F - l;
      const bool eob = is_ac && size == 0 && run != 15;           // EOB / ZRL: jdhuff.c rule
      for (int f = 0; f < (1 << sh); ++f) {
        uint32_t e = kFastValid | (uint32_t)(eob ? 64 : run + 1) << kFastAdvShift;
        if (l + size <= F) {                                        // value fits: decode it here
          const int bits = size ? (f >> (sh - size)) & ((1 << size) - 1) : 0;
          const int v = size ? (bits < (1 << (size - 1)) ? bits - (1 << size) + 1 : bits) : 0;
          e = (e & ~0xFFFFu) | kFastFull | (uint32_t)(l + size) << 25 | (uint32_t)(uint16_t)(int16_t)v;
        } else {
          e |= (uint32_t)l << 25 | (uint32_t)size;
        }
        o->fast[(code << sh) | f] = e;
      }
    }
    if (code >= (1 << l)) return false;   // over-subscribed or an all-ones code (jdhuff.c rule)
    code <<= 1;
  }
  o->maxcode[17] = 0x7fffffff;
  if (k != t.nvals) return false;
  std::memcpy(o->vals, t.vals, k);
  o->is_ac = is_ac ? 1 : 0;
  return true;
}

}  // namespace bbx
