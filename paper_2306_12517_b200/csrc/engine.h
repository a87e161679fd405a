// Host-side declarations of libbbx (C++17).  The C ABI is in include/bbx.h.
#pragma once
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bbx_internal.h"

namespace bbx {

// ---- errors: thread-local message + status code (errors.py classes)
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
const char* last_error();

#define CK(expr)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return ::bbx::fail(BBX_CUDA_ERROR, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                               \
  } while (0)

// ---- rng.py:23-79
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
inline uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
inline uint64_t fold(uint64_t s, uint64_t v) { return mix64(s + kGolden + v); }
struct Rng {
  uint64_t state;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next() { state += kGolden; return mix64(state); }
  uint64_t below(uint64_t n) { return next() % n; }
  bool chance(double p) {
    if (p <= 0.0) return false;
    if (p >= 1.0) return true;
    return next() < (uint64_t)(p * 18446744073709551616.0);
  }
  double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// ---- dataset
struct Field {
  bbx_field_info info;
  int cell_width = 0;
  int64_t array_nbytes = 0;
};
struct ImageCell {
  uint64_t offset, length;
  int h, w, c, codec;
};

}  // namespace bbx

struct bbx_dataset {
  std::string path;
  int fd = -1;
  const uint8_t* map = nullptr;
  size_t map_len = 0;
  int64_t num_samples = 0, page_size = 0, data_table_offset = 0, heap_offset = 0, alloc_table_offset = 0;
  int row_width = 0;
  std::vector<bbx::Field> fields;
  const uint8_t* rows = nullptr;
  int resident_device = -1;
  uint8_t* d_heap = nullptr;   // device copy of [heap_offset, alloc_table_offset)
  bool populated = false;        // the mmap's page tables were filled in (staged loaders, engine.cpp finalize)
  uint8_t* h_heap = nullptr;     // pinned host copy of the heap (bbx_dataset_pin_host)
  uint8_t* h_heap_dev = nullptr; // its device-mapped address (zero-copy reads over PCIe)
  std::mutex reg_mu;
  ~bbx_dataset() {
    if (map) munmap((void*)map, map_len);
    if (fd >= 0) ::close(fd);
  }
};

namespace bbx {
int dataset_open(const char* path, bbx_dataset** out);
void dataset_close(bbx_dataset* ds);
int dataset_make_resident(bbx_dataset* ds, int device);
int dataset_pin_host(bbx_dataset* ds, int threads);
ImageCell image_cell(const bbx_dataset* ds, int64_t i, const Field& f);
uint64_t u64_cell(const bbx_dataset* ds, int64_t i, const Field& f);
int64_t primary_page(const bbx_dataset* ds, int64_t i);

int epoch_order(int kind, uint64_t seed, uint64_t epoch, int64_t n, const int64_t* page_map, int64_t batch_size,
                int64_t* out);

// RandomResizedCrop / CenterCrop windows (extension decoders).
void rrc_window(Rng& r, int h, int w, const double scale[2], const double ratio[2], int* top, int* left, int* ch,
                int* cw, const double* log_ratio = nullptr);
void center_window(int h, int w, double ratio, int* top, int* left, int* ch, int* cw);

// ---- fixed-size worker pool for payload gathers
class Pool {
 public:
  explicit Pool(int n);
  ~Pool();
  // Runs fn(i) for i in [0, n) on the pool (and the caller); returns when done.
  // fn(0) .. fn(n - 1) on the workers and the caller; indices are claimed `grain` at a
  // time (tiny items: one shared-counter round trip per item costs more than the item)
  void parallel_for(int64_t n, const std::function<void(int64_t)>& fn, int64_t grain = 1);
  int size() const { return (int)workers_.size() + 1; }
  // Restrict the worker threads to `cpus` (NUMA placement of the staging gather).
  void pin(const std::vector<int>& cpus);

 private:
  // One parallel_for call.  Each call owns its counters, so a worker that wakes
  // late for an earlier call can neither run that call's function again nor
  // claim indices of the next call (workers hold a shared_ptr to the job).
  struct Job {
    const std::function<void(int64_t)>* fn = nullptr;
    int64_t n = 0, grain = 1;
    alignas(64) std::atomic<int64_t> next{0};   // claimed by every worker
    alignas(64) std::atomic<int64_t> done{0};   // polled by the caller
  };
  void run();
  void work(Job& job);
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Job> job_;
  std::atomic<uint64_t> gen_{0};   // bumped per job; spinning workers poll it without the lock
  bool stop_ = false;
};

}  // namespace bbx
