// Epoch orders (traversal.py:45-120) and the extension crop windows, native.
//
// QUASI_RANDOM is O(N log P) here instead of the reference's O(N*B) list
// walk, but draw-for-draw identical: a Fenwick tree over admission slots
// finds the k-th unconsumed sample in admission order, and each page's list
// keeps its order under pop(k) (traversal.py:64-72).
#include <algorithm>
#include <cmath>
#include <map>

#include "engine.h"

namespace bbx {

int epoch_order(int kind, uint64_t seed, uint64_t epoch, int64_t n, const int64_t* page_map, int64_t batch_size,
                int64_t* out) {
  if (n < 0) return fail(BBX_INVALID_ARGUMENT, "num_samples must be >= 0");
  if (kind == 0) {                                       // SEQUENTIAL
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    return BBX_OK;
  }
  Rng r(fold(fold(seed, 1), epoch));                     // stream_seed(seed, TAG_ORDER, epoch)
  if (kind == 1) {                                       // RANDOM: Rng.shuffle (rng.py:75-79)
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    for (int64_t i = n - 1; i > 0; --i) {
      int64_t j = (int64_t)r.below((uint64_t)(i + 1));
      std::swap(out[i], out[j]);
    }
    return BBX_OK;
  }
  if (kind != 2) return fail(BBX_INVALID_ARGUMENT, "unknown order kind %d", kind);
  if (batch_size < 1) return fail(BBX_INVALID_ARGUMENT, "quasi-random order requires batch_size >= 1");
  if (n == 0) return BBX_OK;
  // by_page in sample order; pages sorted ascending with None (-1) last
  std::map<int64_t, std::vector<int64_t>> by_page;
  std::vector<int64_t> none;
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = page_map ? page_map[i] : -1;
    if (p < 0) none.push_back(i); else by_page[p].push_back(i);
  }
  std::vector<std::vector<int64_t>*> order;
  for (auto& kv : by_page) order.push_back(&kv.second);
  if (!none.empty()) order.push_back(&none);
  const int64_t P = (int64_t)order.size();
  for (int64_t i = P - 1; i > 0; --i) {                  // r.shuffle(page_order)
    int64_t j = (int64_t)r.below((uint64_t)(i + 1));
    std::swap(order[i], order[j]);
  }
  // Fenwick tree over admission slot (== position in page order) -> remaining count
  std::vector<int64_t> fw(P + 1, 0);
  auto add = [&](int64_t i, int64_t v) { for (++i; i <= P; i += i & -i) fw[i] += v; };
  int64_t logp = 1;
  while ((logp << 1) <= P) logp <<= 1;
  auto kth = [&](int64_t k) {                            // smallest slot with prefix > k
    int64_t pos = 0;
    for (int64_t step = logp; step; step >>= 1)
      if (pos + step <= P && fw[pos + step] <= k) { pos += step; k -= fw[pos]; }
    return std::make_pair(pos, k);                       // slot index, offset within it
  };
  std::vector<std::vector<int64_t>> lists(P);
  int64_t admitted = 0, next_page = 0, total = 0, emitted = 0;
  while (emitted < n) {
    while (admitted < batch_size && next_page < P) {    // eager refill (traversal.py:57-63)
      lists[next_page] = *order[next_page];
      add(next_page, (int64_t)lists[next_page].size());
      total += (int64_t)lists[next_page].size();
      ++next_page; ++admitted;
    }
    uint64_t k = r.below((uint64_t)total);
    auto [slot, off] = kth((int64_t)k);
    auto& L = lists[slot];
    out[emitted++] = L[off];
    L.erase(L.begin() + off);                            // samples.pop(k)
    add(slot, -1);
    --total;
    if (L.empty()) --admitted;                           // admitted.pop(slot)
  }
  return BBX_OK;
}

// RandomResizedCrop window (extension).  The rule of torchvision /
// FFCV get_random_crop with bbox Rng draws; identical expression order to
// oracle/bbx_oracle.c:or_rrc_window so the same libm gives the same window.
void rrc_window(Rng& r, int h, int w, const double scale[2], const double ratio[2], int* top, int* left, int* ch,
                int* cw, const double* log_ratio) {
  double area = (double)h * (double)w;
  // log(ratio) is a per-op constant: the loader passes it precomputed (same libm value)
  double lr0 = log_ratio ? log_ratio[0] : std::log(ratio[0]), lr1 = log_ratio ? log_ratio[1] : std::log(ratio[1]);
  for (int attempt = 0; attempt < 10; ++attempt) {
    double target = area * (scale[0] + (scale[1] - scale[0]) * r.uniform());
    double aspect = std::exp(lr0 + (lr1 - lr0) * r.uniform());
    int ww = (int)std::nearbyint(std::sqrt(target * aspect));
    int hh = (int)std::nearbyint(std::sqrt(target / aspect));
    if (ww > 0 && ww <= w && hh > 0 && hh <= h) {
      *top = (int)r.below((uint64_t)(h - hh + 1));
      *left = (int)r.below((uint64_t)(w - ww + 1));
      *ch = hh; *cw = ww;
      return;
    }
  }
  double in_ratio = (double)w / (double)h;
  int ww, hh;
  if (in_ratio < ratio[0]) { ww = w; hh = (int)std::nearbyint(ww / ratio[0]); }
  else if (in_ratio > ratio[1]) { hh = h; ww = (int)std::nearbyint(hh * ratio[1]); }
  else { ww = w; hh = h; }
  hh = std::min(std::max(hh, 1), h);
  ww = std::min(std::max(ww, 1), w);
  *top = (h - hh) / 2; *left = (w - ww) / 2; *ch = hh; *cw = ww;
}

void center_window(int h, int w, double ratio, int* top, int* left, int* ch, int* cw) {
  int s = std::min(h, w);
  int c = std::max((int)(ratio * (double)s), 1);
  *top = (h - c) / 2; *left = (w - c) / 2; *ch = c; *cw = c;
}

}  // namespace bbx
