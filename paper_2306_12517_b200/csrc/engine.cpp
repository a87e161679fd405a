// The batch-granular device loader behind bbx_loader_* (include/bbx.h).
//
// Replaces the reference's per-sample worker machinery (loader.py:251-447:
// _EpochRun, FillState, _process_position; pipeline.py:302-406 PipelinePlan)
// with one pipeline per loader:
//
//   submit(slot, idx)  ->  [pipeline thread]
//        1. host: rows -> per-sample descriptors + RNG params (rng.py, exact),
//           payload checks with the reference's error texts (codecs.py:91-128)
//        2. pool threads gather payload extents mmap -> pinned staging slot
//        3. copy stream: one cudaMemcpyAsync H2D of the whole slot
//        4. compute stream: K2 RLE expand (if any RLE sample), K1/K3 kernels,
//           status D2H; record slot `done` event
//   wait(slot)         ->  cudaEventSynchronize(done) + error merge
//
// Slots are double/triple buffered: the gather of batch g+2 overlaps the H2D
// of g+1 and the kernels of g.  With a device-resident heap
// (bbx_dataset_make_resident) steps 2-3 shrink to the descriptor upload.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <unordered_map>
#include <deque>
#include <set>

#include "engine.h"
#include "jpeg.h"

namespace bbx {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
const char* last_error() { return g_err.c_str(); }

// -------------------------------------------------------------------- pool
Pool::Pool(int n) {
  for (int i = 0; i < n - 1; ++i) workers_.emplace_back([this] { run(); });
}
Pool::~Pool() {
  { std::lock_guard<std::mutex> g(mu_); stop_ = true; }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}
static bool set_affinity(pthread_t th, const std::vector<int>& cpus) {
  if (cpus.empty()) return false;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus) if (c >= 0 && c < CPU_SETSIZE) CPU_SET(c, &set);
  return pthread_setaffinity_np(th, sizeof set, &set) == 0;
}
void Pool::pin(const std::vector<int>& cpus) {
  for (auto& t : workers_) set_affinity(t.native_handle(), cpus);
}

// NUMA placement.  The CPUs of the GPU's NUMA node (sysfs: the
// PCI device's numa_node, the node's cpulist) that this process may run on;
// with several ranks per node (torchrun LOCAL_RANK / LOCAL_WORLD_SIZE, GPUs
// spread evenly over the nodes) each rank takes its own slice of them.
// Empty when the topology is unknown (the threads then float).
static std::vector<int> parse_cpulist(const std::string& s) {
  std::vector<int> out;
  size_t i = 0;
  while (i < s.size()) {
    char* end = nullptr;
    const long a = std::strtol(s.c_str() + i, &end, 10);
    if (end == s.c_str() + i) break;
    long b = a;
    i = (size_t)(end - s.c_str());
    if (i < s.size() && s[i] == '-') { b = std::strtol(s.c_str() + i + 1, &end, 10); i = (size_t)(end - s.c_str()); }
    for (long c = a; c <= b; ++c) out.push_back((int)c);
    while (i < s.size() && (s[i] == ',' || s[i] == '\n' || s[i] == ' ')) ++i;
  }
  return out;
}
static std::string read_small(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) return "";
  char buf[4096];
  const size_t n = std::fread(buf, 1, sizeof buf - 1, f);
  std::fclose(f);
  buf[n] = 0;
  return buf;
}
static std::vector<int> gpu_local_cpus(int device, int* node_out) {
  *node_out = -1;
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) { cudaGetLastError(); return {}; }
  std::string id(bus);
  for (auto& ch : id) ch = (char)std::tolower((unsigned char)ch);
  const std::string ns = read_small("/sys/bus/pci/devices/" + id + "/numa_node");
  if (ns.empty()) return {};
  const int node = std::atoi(ns.c_str());
  if (node < 0) return {};
  *node_out = node;
  std::vector<int> cpus = parse_cpulist(read_small("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"));
  cpu_set_t allowed;
  if (sched_getaffinity(0, sizeof allowed, &allowed) == 0)
    cpus.erase(std::remove_if(cpus.begin(), cpus.end(), [&](int c) { return c >= CPU_SETSIZE || !CPU_ISSET(c, &allowed); }),
               cpus.end());
  int nodes = 0;
  for (int k = 0; k < 64; ++k)
    if (!read_small("/sys/devices/system/node/node" + std::to_string(k) + "/cpulist").empty()) ++nodes;
  const char* lws = std::getenv("LOCAL_WORLD_SIZE");
  const char* lr = std::getenv("LOCAL_RANK");
  if (lws && lr && nodes > 0 && !cpus.empty()) {
    const int per_node = std::max(1, std::atoi(lws) / nodes), slice = std::atoi(lr) % per_node;
    const size_t n = cpus.size() / (size_t)per_node;
    if (n > 0) cpus = std::vector<int>(cpus.begin() + (size_t)slice * n, cpus.begin() + (size_t)(slice + 1) * n);
  }
  return cpus;
}

void Pool::work(Job& job) {
  const int64_t g = job.grain;
  for (int64_t i; (i = job.next.fetch_add(g)) < job.n;) {
    const int64_t e = std::min(job.n, i + g);
    for (int64_t k = i; k < e; ++k) (*job.fn)(k);
    if (job.done.fetch_add(e - i) + (e - i) == job.n) {
      std::lock_guard<std::mutex> g(mu_);
      done_cv_.notify_all();
    }
  }
}
// A worker that just finished a job polls for the next one for a short while before
// sleeping on the condition variable: batches arrive every few tens of microseconds,
// and a futex wake-up costs about as much as a batch's descriptor work.
static constexpr auto kPoolSpin = std::chrono::microseconds(60);
static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#endif
}
void Pool::run() {
  uint64_t seen = 0;
  for (;;) {
    const auto until = std::chrono::steady_clock::now() + kPoolSpin;
    while (gen_.load(std::memory_order_acquire) == seen && std::chrono::steady_clock::now() < until) cpu_relax();
    std::shared_ptr<Job> job;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_.load() != seen; });
      if (stop_) return;
      seen = gen_.load();
      job = job_;
    }
    if (job) work(*job);
  }
}
void Pool::parallel_for(int64_t n, const std::function<void(int64_t)>& fn, int64_t grain) {
  if (n <= 0) return;
  if (workers_.empty() || n == 1) { for (int64_t i = 0; i < n; ++i) fn(i); return; }
  auto job = std::make_shared<Job>();
  job->fn = &fn;
  job->n = n;
  job->grain = std::max<int64_t>(1, grain);
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = job;
    gen_.fetch_add(1, std::memory_order_release);
  }
  cv_.notify_all();
  work(*job);
  // the caller's share is done: poll the stragglers briefly, then sleep
  const auto until = std::chrono::steady_clock::now() + kPoolSpin;
  while (job->done.load(std::memory_order_acquire) < n && std::chrono::steady_clock::now() < until) cpu_relax();
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return job->done.load() >= n; });
  if (job_ == job) job_.reset();
}

// -------------------------------------------------------------------- plan
static int dtype_size(int dt) {
  switch (dt) { case BBX_U8: return 1; case BBX_I64: case BBX_F64: return 8; case BBX_F32: return 4; default: return 2; }
}
static uint16_t f32_to_bf16_bits(float f) {      // round to nearest even
  uint32_t u; std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static uint16_t f32_to_f16_bits(float f) {       // IEEE binary16, round to nearest even
  uint32_t x; std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u, ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) return (uint16_t)(sign | (ax > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);            // rounds to inf
  if (ax < 0x38800000u) {                                                // half subnormal
    if (ax < 0x33000000u) return (uint16_t)sign;                         // <= 2^-25 ties to 0
    uint32_t mant = (ax & 0x7fffffu) | 0x800000u;
    int shift = 126 - (int)(ax >> 23) + 14;
    uint32_t q = mant >> shift, rem = mant & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return (uint16_t)(sign | q);
  }
  uint32_t r = ax - 0x38000000u, q = r >> 13, rem = r & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;
  return (uint16_t)(sign | q);
}

struct Draw {        // one RNG-consuming op, in chain order (host program)
  int kind;          // BBX_OP_RRC / BBX_OP_CENTERCROP / BBX_OP_CROP / BBX_OP_FLIP
  int slot;          // first param slot
  int in_h, in_w, h, w;
  double p;
  double scale[2], ratio[2];
  double log_ratio[2];   // RRC: log(ratio), computed once at plan time
};

struct Plan {
  int field_index = -1;
  bool scalar = false;
  PlanDev dev{};
  std::vector<Draw> draws;
  int64_t out_sample_bytes = 0;
  int64_t max_payload = 0;       // over the whole dataset (exact staging capacity)
  bool field_has_rle = false;
  bool field_has_jpeg = false;
  int64_t jpeg_blocks_cap = 0;   // per sample: coefficient blocks (any sampling with factors <= 2)
  int64_t jpeg_int_cap = 0;      // per sample: restart intervals (<= MCUs)
  // per compute stream (batches alternate between kStreams streams; one stream orders its own)
  int16_t* d_coef[kStreams] = {};           // JPEG coefficients
  uint8_t* d_planes[kStreams] = {};         // IDCT output: component planes
  unsigned long long* d_ticket[kStreams] = {};   // column-walker K1 tile ticket (2 x u64, zero between launches)
  void* d_lut = nullptr;
  std::vector<void*> outs;       // per slot
  std::vector<uint8_t*> d_scratch;
  std::vector<uint32_t*> d_tables;   // per slot: K1 prologue tables
  std::vector<JpegDesc> jcache;      // per sample, valid where jcached[i] (JPEG fields)
  std::vector<std::vector<uint32_t>> jstarts;   // per sample: first byte of each restart interval
  std::vector<uint8_t> jcached;
  uint64_t* d_col = nullptr;     // scalar column (num_samples x 8 B)
};

struct HostErr { int64_t pos = -1; int plan = 0; int code = 0; std::string msg; };

struct Slot {
  uint8_t* h_stage = nullptr;
  uint8_t* d_stage = nullptr;
  int n_gcopies = 0;                  // zero-copy gather: payload copies the device gathers for this batch
  size_t cap = 0;
  SampleStatus* d_status = nullptr;
  SampleStatus* h_status = nullptr;
  cudaEvent_t h2d_done{}, done{}, release{};
  cudaEvent_t h2d_t{};             // profiling: timed copy of h2d_done
  bool h2d_timed = false;
  bool h2d_on_compute = false;     // the last H2D ran on the batch's compute stream (no h2d_done record)
  cudaGraphExec_t gexec[kStreams] = {};   // the slot's captured batch per compute stream (resident, full batch)
  int glaunches[kStreams] = {};           // kernels in that graph
  int last_stream = -1;            // compute stream of the slot's last batch
  cudaEvent_t k0{}, k1{};          // profiling: around the transform kernels
  bool timed = false;
  int64_t timed_launches = 0, timed_bytes = 0;
  bool released_pending = false, used = false;
  uint64_t serial = 0;             // batches this ring slot has launched (page-pool reuse guards)
  // job
  int state = 0;                 // 0 idle, 1 queued, 2 launched
  int count = 0;
  uint64_t seed = 0, epoch = 0;
  std::vector<int64_t> idx;
  HostErr herr;
  int fatal = 0;
  std::string fatal_msg;
  std::vector<char> plan_has_rle;
  std::vector<char> plan_has_jpeg;
  std::vector<uint32_t> jpeg_total_int;
  std::vector<uint64_t> jpeg_total_blk;
  std::vector<int32_t> jpeg_max_quads;
  std::vector<uint32_t> jpeg_max_blocks;
};

// Device pools of the Huffman / quant tables the JPEG samples reference,
// deduplicated by content (one writer's files share a handful).  Append-only:
// entries in use by in-flight kernels never change.
struct JpegTables {
  JHuff* h_huff = nullptr;       // pinned host mirrors
  JQuant* h_quant = nullptr;
  JHuff* d_huff = nullptr;
  JQuant* d_quant = nullptr;
  int n_huff = 0, n_quant = 0, up_huff = 0, up_quant = 0;
  // content hash -> ids (several on a collision); raw bytes kept to verify
  std::unordered_multimap<uint64_t, int> hmap, qmap;
  std::vector<std::vector<uint8_t>> hkey, qkey;
  std::mutex mu;                 // headers are parsed on the staging pool
};

// One epoch's page plan (reader.py:96-145 PageSchedule over the trace loader.py:
// 276-291 builds): the batches' samples, and per batch its trace positions
// (the distinct heap pages of each sample, ascending) with the plan's fetch /
// eviction steps.  An eviction whose victim this same batch already used is
// "deferred": the batch's kernels read every page of the batch at once, so
// the victim's buffer is recycled after them (a spare physical page slot
// holds the incoming page meanwhile).
struct PageStep {
  int64_t page;
  int64_t victim;      // -1: no eviction
  uint8_t fetch, deferred, reload;
};
struct PagePlan {
  std::vector<int64_t> idx;           // samples, batch after batch
  std::vector<int64_t> batch_off;     // first sample of batch b in idx (n_batches + 1 entries)
  std::vector<int64_t> trace_off;     // first trace position of sample k (idx.size() + 1 entries)
  std::vector<PageStep> trace;
  int64_t phys_needed = 0;            // capacity + most deferred evictions of one batch
  int64_t fetches = 0, reloads = 0;
  int32_t next = 0;                   // next batch to execute
};
constexpr int kPageBufs = 4;          // pinned host page buffers (fetch staging)
struct PagePool {
  int64_t capacity = 0;               // capacity_pages (0: no page pool)
  double fetch_latency_s = 0.0;       // reader.py ProcessCache fetch_latency_s (spin before each fetch)
  int64_t phys = 0;                   // physical page slots allocated in d_pool
  uint8_t* d_pool = nullptr;
  std::deque<PagePlan> plans;         // installed epochs, executed in submission order (bbx_loader_plan_epoch)
  std::vector<int64_t> slot_of;       // heap page -> physical slot (-1: not resident)
  std::vector<int64_t> page_in;       // physical slot -> heap page (-1: free)
  std::vector<int32_t> user_ring;     // physical slot -> ring slot of the last batch that read it (-1: none)
  std::vector<uint64_t> user_serial;  //   ... and that batch's serial (the ring slot's, at submission)
  std::vector<int64_t> free_list;
  uint8_t* h_buf = nullptr;           // kPageBufs x page_size pinned
  cudaEvent_t buf_ev[kPageBufs]{};
  bool buf_used[kPageBufs] = {};
  int buf_next = 0;
};

}  // namespace bbx

using namespace bbx;

struct bbx_loader {
  bbx_dataset* ds = nullptr;
  int device = 0;
  int batch = 0, nslots = 0;
  std::vector<Plan> plans;
  std::vector<Slot> slots;
  cudaStream_t copy_st{}, comp_st[kStreams]{};   // batches alternate between the compute streams
  uint64_t batch_seq = 0;             // batches launched (pipeline thread): picks the stream
  int nstreams = kStreams;            // compute streams in use (option "compute_streams": 1 or 2)
  std::unique_ptr<Pool> pool;
  bool finalized = false;
  size_t slot_bytes = 0, desc_bytes = 0, idx_off = 0;
  std::vector<size_t> desc_off;       // per plan, within a slot
  std::vector<size_t> jpeg_off;       // per plan with JPEG samples: JpegDesc[B] + prefixes, within a slot
  JpegTables jt;
  bool jpeg_cache = true;             // keep each sample's prepared JpegDesc (headers parse once per loader)
  bool jpeg_roi = true;               // decode only the MCUs a sample's chain reads (BBX_JPEG_ROI=0: whole image)
  bool jpeg_prefetch = true;          // parse headers at finalize (file fits in RAM; option "jpeg_header_prefetch" 0: lazily)
  std::vector<int64_t> prefetch_set;  // samples whose headers finalize parses (empty: every sample)
  bool zero_copy = false;             // requested: kernels read payloads from the pinned host heap
  const uint8_t* payload_dev = nullptr;   // set at finalize: HBM heap, mapped pinned heap, or null (staging)
  bool zc = false;                    // payload_dev is host memory (zero-copy)
  bool zc_gather = true;              // zero-copy heap: a gather kernel stages the batch's rows (option "zc_gather")
  bool zcg = false;                   // set at finalize: zero-copy gather in use
  size_t gcopy_off = 0;               // GatherCopy list within a slot (zero-copy gather)
  size_t pay_base = 0;                // start of the compact payload region
  bool window_staging = true;         // stage only the rows/columns a RAW sample's chain reads
  int64_t par_desc_min = 256;         // batches of at least this many samples fill descriptors on the pool
  bool use_graphs = true;             // replay full resident batches as CUDA graphs (option "cuda_graphs")
  std::vector<int> local_cpus;        // the GPU's NUMA-node CPUs (this rank's slice); empty: unknown
  int numa_node = -1;
  bool direct_io = false;             // Direct strategy (reader.py:61-65,368-372): one pread per payload read
  int64_t read_latency_ns = 0;        //   ... with the strategy's read latency spun before each read
  // HBM page pool (ProcessCacheStrategy with capacity < num_pages): executes the
  // reference's Belady PageSchedule (reader.py:96-145) batch by batch
  PagePool pp;
  // pipeline thread
  std::thread th;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::deque<int> queue;
  bool stop = false;
  bbx_loader_stats stats{};
  bool profiling = false;
  int prof_every = 1;                // profile every n-th batch (bbx_loader_set_profiling(n))
  uint64_t prof_seq = 0;
  cudaEvent_t t_ref{};               // profiling: reference for absolute batch times (idle gaps)
  float last_k1_ms = -1.f;
  std::mutex stats_mu;
};

namespace bbx {

// The kernel's divide-free normalize (kernels.cu: apply_vops_fma) must equal
// the IEEE quotient bit for bit; a u8 plan has only 256 inputs per channel,
// so prove it by enumeration (host fma == device fma: both correctly rounded).
static bool verify_fma_normalize(const PlanDev& P, int C) {
  for (int k = 0; k < std::min(C, 4); ++k)
    for (int v = 0; v < 256; ++v) {
      float x = (float)v, y = (float)v;
      for (int i = 0; i < P.n_vops; ++i) {
        volatile float t = x - P.vop_mean[i][k];
        x = t / P.vop_std[i][k];
        volatile float dd = y - P.vop_mean[i][k];
        float d = dd;
        volatile float q0v = d * P.vop_inv[i][k];
        float q0 = q0v;
        float r = std::fma(-q0, P.vop_std[i][k], d);
        y = std::fma(r, P.vop_inv[i][k], q0);
        if (std::memcmp(&x, &y, 4) != 0) return false;
      }
    }
  return true;
}

// f16 / bf16 output of a u8 value chain through the column-walker K1: the
// kernel forms y = fma(u, A_c, B_c) in f32 and rounds it to the output type
// (cvt.rn.f16x2 / bf16x2).  The chain (x - m) / s ... is affine in u; the
// coefficients are searched a few ulps around their double-precision values
// until the result equals the exact value table (`lut`, the reference's IEEE
// subtract + divide, pipeline.py:158-160) for every one of the 256 inputs of
// every channel -- a proof by enumeration, as verify_fma_normalize.  No pair
// found: the kernel keeps the table.
static bool prove_affine(PlanDev& P, int C, const std::vector<uint8_t>& lut, int out_dt) {
  for (int k = 0; k < C; ++k) {
    double a = 1.0, b = 0.0;
    for (int i = 0; i < P.n_vops; ++i) {
      a = a / P.vop_std[i][k];
      b = (b - P.vop_mean[i][k]) / P.vop_std[i][k];
    }
    const uint16_t* want = reinterpret_cast<const uint16_t*>(lut.data()) + (size_t)k * 256;
    auto ok = [&](float A, float B) {
      for (int v = 0; v < 256; ++v) {
        const float y = std::fma((float)v, A, B);
        const uint16_t got = out_dt == BBX_F16 ? f32_to_f16_bits(y) : f32_to_bf16_bits(y);
        if (got != want[v]) return false;
      }
      return true;
    };
    bool found = false;
    const float A0 = (float)a, B0 = (float)b;
    float A = A0;
    for (int da = 0; da <= 8 && !found; ++da) {
      for (int sa = 0; sa < (da ? 2 : 1) && !found; ++sa) {
        A = A0;
        for (int i = 0; i < da; ++i) A = std::nextafter(A, sa ? -INFINITY : INFINITY);
        for (int db = 0; db <= 32 && !found; ++db)
          for (int sb = 0; sb < (db ? 2 : 1) && !found; ++sb) {
            float B = B0;
            for (int i = 0; i < db; ++i) B = std::nextafter(B, sb ? -INFINITY : INFINITY);
            if (ok(A, B)) { P.cw_aff_a[k] = A; P.cw_aff_b[k] = B; found = true; }
          }
      }
    }
    if (!found) return false;
  }
  for (int v = 0; v < 6; ++v) { P.cw_pair_a[v] = P.cw_aff_a[v % 3]; P.cw_pair_b[v] = P.cw_aff_b[v % 3]; }
  return true;
}

static int host_back_y(const PlanDev& P, const int32_t* prm, int y);

// Integer bilinear axis rule (kernel lin_axis / oracle lin_axis), host copy.
static void host_lin_axis(int o, int out_n, int in_n, int* i0, int* i1) {
  int64_t num = (int64_t)(2 * o + 1) * in_n - out_n, den = 2 * (int64_t)out_n;
  if (num <= 0) { *i0 = 0; *i1 = 0; return; }
  int64_t q = num / den;
  if (q >= in_n - 1) { *i0 = in_n - 1; *i1 = in_n - 1; return; }
  *i0 = (int)q; *i1 = (int)q + 1;
}

static int plan_compile(bbx_loader* L, int field_index, const bbx_op* ops, int n_ops, Plan& pl) {
  const bbx_dataset* ds = L->ds;
  if (field_index < 0 || field_index >= (int)ds->fields.size())
    return fail(BBX_INVALID_ARGUMENT, "field index %d out of range", field_index);
  const Field& f = ds->fields[field_index];
  if (n_ops < 1) return fail(BBX_SPEC_MISMATCH, "a pipeline needs at least one transform");
  PlanDev& P = pl.dev;
  std::memset(&P, 0, sizeof P);
  pl.field_index = field_index;
  int H, W, C, dt, ndim;
  int nparams = 0;
  const bbx_op& s0 = ops[0];
  if (s0.kind == BBX_OP_DECODE || s0.kind == BBX_OP_RRC || s0.kind == BBX_OP_CENTERCROP) {
    if (f.info.kind != 4) return fail(BBX_SPEC_MISMATCH, "decode expects an image field, got field '%s'", f.info.name);
    C = f.info.channels;
    P.src_row_w = f.info.max_width;
    if (s0.kind == BBX_OP_DECODE) {
      P.src_kind = SRC_DECODE; H = f.info.max_height; W = f.info.max_width;
    } else {
      if (s0.h < 1 || s0.w < 1) return fail(BBX_SPEC_MISMATCH, "decoder output size must be >= 1");
      P.src_kind = SRC_RESAMPLE; H = s0.h; W = s0.w;
      Draw d{}; d.kind = s0.kind; d.slot = 0; d.h = s0.h; d.w = s0.w; d.p = s0.p;
      d.scale[0] = s0.scale[0]; d.scale[1] = s0.scale[1]; d.ratio[0] = s0.ratio[0]; d.ratio[1] = s0.ratio[1];
      d.log_ratio[0] = std::log(d.ratio[0]); d.log_ratio[1] = std::log(d.ratio[1]);
      if (s0.kind == BBX_OP_RRC && !(d.scale[0] > 0 && d.scale[0] <= d.scale[1] && d.ratio[0] > 0 && d.ratio[0] <= d.ratio[1]))
        return fail(BBX_SPEC_MISMATCH, "random-resized-crop needs 0 < scale[0] <= scale[1] and 0 < ratio[0] <= ratio[1]");
      if (s0.kind == BBX_OP_CENTERCROP && !(d.p > 0 && d.p <= 1.0))
        return fail(BBX_SPEC_MISMATCH, "center-crop ratio must be in (0, 1]");
      pl.draws.push_back(d);
      nparams = 4;
    }
    dt = BBX_U8; ndim = 3;
    P.src_elem = 1; P.src_dtype = BBX_U8;
  } else if (s0.kind == BBX_OP_ARRAYREAD) {
    if (f.info.kind != 2) return fail(BBX_SPEC_MISMATCH, "array-read expects an array field, got field '%s'", f.info.name);
    static const int map_dt[4] = {BBX_U8, BBX_I64, BBX_F32, BBX_F64};
    dt = map_dt[f.info.array_dtype];
    ndim = f.info.ndims;
    P.src_kind = SRC_ARRAY; P.src_elem = dtype_size(dt); P.src_dtype = dt;
    if (ndim == 3) { H = (int)f.info.dims[0]; W = (int)f.info.dims[1]; C = (int)f.info.dims[2]; }
    else {
      int64_t last = f.info.dims[ndim - 1], tot = 1;
      for (int k = 0; k < ndim; ++k) tot *= f.info.dims[k];
      if (tot > INT32_MAX) return fail(BBX_SPEC_MISMATCH, "array field too large for a device plan");
      H = 1; W = (int)(tot / last); C = (int)last;
    }
    P.src_row_w = W;
  } else {
    return fail(BBX_SPEC_MISMATCH, "the first transform must read from the sample source");
  }
  P.canvas_h = H; P.canvas_w = W; P.channels = C;
  int out_dt = dt;
  bool cast_seen = false;
  for (int i = 1; i < n_ops; ++i) {
    const bbx_op& o = ops[i];
    if (cast_seen) return fail(BBX_SPEC_MISMATCH, "cast must be the last transform");
    switch (o.kind) {
      case BBX_OP_DECODE: case BBX_OP_ARRAYREAD: case BBX_OP_RRC: case BBX_OP_CENTERCROP:
        return fail(BBX_SPEC_MISMATCH, "source transforms may only appear first");
      case BBX_OP_TOFLOAT: case BBX_OP_NORMALIZE: case BBX_OP_NORMALIZE_PC: {
        if (P.n_vops >= kMaxValueOps) return fail(BBX_SPEC_MISMATCH, "too many value transforms");
        if (o.kind == BBX_OP_NORMALIZE_PC && C > 4)
          return fail(BBX_SPEC_MISMATCH, "per-channel normalize supports at most 4 channels");
        out_dt = BBX_F32;
        if (o.kind == BBX_OP_TOFLOAT) break;     // u8/int -> f32 is implicit in every value op
        int v = P.n_vops++;
        for (int k = 0; k < 4; ++k) {             // scalar Normalize is replicated per channel
          int kk = o.kind == BBX_OP_NORMALIZE ? 0 : k;
          P.vop_mean[v][k] = o.mean[kk];
          P.vop_std[v][k] = o.std[kk];
          if (o.kind == BBX_OP_NORMALIZE_PC && k >= C) { P.vop_mean[v][k] = 0.f; P.vop_std[v][k] = 1.f; }
          if (P.vop_std[v][k] == 0.f) return fail(BBX_SPEC_MISMATCH, "normalize std must be nonzero");
          volatile float one = 1.0f;
          P.vop_inv[v][k] = one / P.vop_std[v][k];
        }
        break;
      }
      case BBX_OP_CAST:
        if (o.dtype != BBX_F32 && o.dtype != BBX_F16 && o.dtype != BBX_BF16)
          return fail(BBX_SPEC_MISMATCH, "cast target must be float32, float16 or bfloat16");
        if (out_dt != BBX_F32) return fail(BBX_SPEC_MISMATCH, "cast expects float32 input");
        out_dt = o.dtype; cast_seen = true;
        break;
      case BBX_OP_FLIP: case BBX_OP_CROP: case BBX_OP_RESIZE: {
        if (ndim != 3) return fail(BBX_SPEC_MISMATCH, "%s expects HxWxC input",
                                   o.kind == BBX_OP_FLIP ? "flip" : (o.kind == BBX_OP_CROP ? "crop" : "resize"));
        if (P.n_remaps >= kMaxRemaps) return fail(BBX_SPEC_MISMATCH, "too many geometric transforms");
        Remap& m = P.remaps[P.n_remaps++];
        m.kind = o.kind; m.in_h = H; m.in_w = W;
        Draw d{}; d.kind = o.kind; d.in_h = H; d.in_w = W;
        if (o.kind == BBX_OP_FLIP) {
          m.out_h = H; m.out_w = W; m.prm = nparams; d.slot = nparams; d.p = o.p; nparams += 1;
          pl.draws.push_back(d);
        } else if (o.kind == BBX_OP_CROP) {
          if (H < o.h || W < o.w || o.h < 1 || o.w < 1)
            return fail(BBX_SPEC_MISMATCH, "cannot crop (%d, %d, %d) to %dx%d", H, W, C, o.h, o.w);
          m.out_h = o.h; m.out_w = o.w; m.prm = nparams; d.slot = nparams; d.h = o.h; d.w = o.w; nparams += 2;
          pl.draws.push_back(d);
          H = o.h; W = o.w;
        } else {
          if (o.h < 1 || o.w < 1) return fail(BBX_SPEC_MISMATCH, "resize target must be >= 1");
          m.out_h = o.h; m.out_w = o.w; m.prm = 0;
          H = o.h; W = o.w;
        }
        break;
      }
      default:
        return fail(BBX_SPEC_MISMATCH, "transform kind %d is not a device transform (Opaque stages cannot run on "
                                       "the device path)", o.kind);
    }
  }
  P.out_h = H; P.out_w = W; P.out_c = C;
  P.out_dtype = out_dt;
  P.n_params = nparams;
  P.desc_stride = (kDescHeader + 4 * nparams + 15) / 16 * 16;
  P.has_remaps_3d = P.n_remaps > 0;
  P.out_sample_elems = (int64_t)H * W * C;
  pl.out_sample_bytes = P.out_sample_elems * dtype_size(out_dt);
  const bool has_values = out_dt != dt || P.n_vops > 0;   // any ToFloat / Normalize / cast
  if (P.src_kind == SRC_ARRAY) {
    P.value_mode = has_values ? VAL_DIRECT : VAL_COPY;
  } else {
    // u8 source: values 0..255 only, so the divide-free normalize can be
    // proven exact for this plan by exhausting its inputs.
    if (has_values && P.n_vops == 0) {          // ToFloat only == Normalize(0, 1), exactly
      for (int k = 0; k < 4; ++k) { P.vop_mean[0][k] = 0.f; P.vop_std[0][k] = 1.f; P.vop_inv[0][k] = 1.f; }
      P.n_vops = 1;
    }
    // C <= 4: the whole value chain u8 -> output is a 256-entry table per
    // channel (one smem load per element), built on the host with the
    // reference's exact arithmetic; wider images use the divide-free form
    // when it is proven exact, else the IEEE divide.
    P.value_mode = !has_values ? VAL_COPY
                 : C <= 4 ? VAL_LUT
                 : verify_fma_normalize(P, C) ? VAL_FMA : VAL_DIRECT;
    if (P.value_mode == VAL_COPY && out_dt != BBX_U8) return fail(BBX_SPEC_MISMATCH, "unexpected output dtype");
    // tile height: 16 rows, shrunk until the smem layout allows 4 CTAs per SM
    P.rows_per_tile = std::min(16, H);
    for (;;) {
      P.lay = img_layout_host(P);
      P.smem_bytes = P.lay.total;
      if (P.smem_bytes <= kSmemTarget || P.rows_per_tile == 1) break;
      P.rows_per_tile = std::max(1, P.rows_per_tile / 2);
    }
    if (P.smem_bytes > kSmemBudget || (int64_t)P.src_row_w * C + 64 > 65535)
      return fail(BBX_SPEC_MISMATCH, "image rows too wide for the device plan (%d x %d channels)", P.src_row_w, C);
    P.tiles_per_sample = (H + P.rows_per_tile - 1) / P.rows_per_tile;
    P.scratch_bytes = (int64_t)f.info.max_height * jpeg_scratch_pitch(f.info.max_width, C);   // RLE: h*w*C <= this
    // fast-division constants (exact when n * d < 2^32)
    const uint64_t two32 = 1ull << 32;
    const int nslot = P.rows_per_tile * (P.src_kind == SRC_RESAMPLE ? 2 : 1);
    if (W > 1 && (uint64_t)nslot * W * W < two32) P.ow_magic = (uint32_t)((two32 + W - 1) / W);
    const int V = 16 / dtype_size(out_dt), gpr = W / V;
    if (gpr > 1 && (uint64_t)P.rows_per_tile * gpr * gpr < two32) P.gpr_magic = (uint32_t)((two32 + gpr - 1) / gpr);
    const uint64_t ax = std::max((uint64_t)H * f.info.max_height, (uint64_t)W * f.info.max_width);
    P.lin32 = 2 * ax < two32 ? 1 : 0;
    if (P.src_kind == SRC_RESAMPLE) {   // lin_axis divides by 2*canvas extent: exact when n*d < 2^32
      auto magic_ok = [&](uint64_t den, uint64_t in_max) {
        return 2048 * den * den < two32 && den * den * in_max < two32;
      };
      uint64_t dx = 2ull * P.canvas_w, dy = 2ull * P.canvas_h;
      if (magic_ok(dx, f.info.max_width)) P.linx_magic = (uint32_t)((two32 + dx - 1) / dx);
      if (magic_ok(dy, f.info.max_height)) P.liny_magic = (uint32_t)((two32 + dy - 1) / dy);
    }
    P.lay = img_layout_host(P);
    P.h_tpc = std::max(1, kThreads / W);
    P.tab_stride = image_tab_stride(P);
    // column-walker K1 for 3-channel bilinear decoders: a compute thread owns
    // two output columns (OW <= 512: at most 8 compute warps), row tags are
    // 16-bit absolute source rows (heights < 0xFFFE)
    P.cw = 0;
    if (P.src_kind == SRC_RESAMPLE && C == 3 && (P.value_mode == VAL_LUT || P.value_mode == VAL_COPY) &&
        W <= 2 * 32 * 8 && f.info.max_height < 0xFFFE) {
      // rows per tile: 16, fewer when a tile could span more than 32 source rows
      for (int rows : {kCwRows, 16, 8, 4, 2}) {
        PlanDev Q = P;
        Q.rows_per_tile = std::min(rows, H);
        Q.tiles_per_sample = (H + Q.rows_per_tile - 1) / Q.rows_per_tile;
        Q.lay = img_layout_host(Q);
        Q.tab_stride = image_tab_stride(Q);
        {   // stage slots: source rows any tile can span.  Rows_per_tile output
            // rows cover at most n canvas rows back through the y remaps, and n
            // canvas rows at most ceil((n - 1) * crop / canvas) + 2 source rows
            // (two taps) with crop <= the field's max height.
          int64_t n = Q.rows_per_tile;
          for (int i = Q.n_remaps - 1; i >= 0; --i)
            if (Q.remaps[i].kind == BBX_OP_RESIZE)
              n = ((n - 1) * Q.remaps[i].in_h + Q.remaps[i].out_h - 1) / Q.remaps[i].out_h + 1;
          const int64_t src = ((n - 1) * f.info.max_height + Q.canvas_h - 1) / Q.canvas_h + 2;
          if (src > 32) continue;
          Q.cw_slots = (int)src;
        }
        Q.cw_npair = (W + 1) / 2;
        Q.cw_warps = (Q.cw_npair + 31) / 32;
        Q.cw_run = kCwRun;
        Q.cw_smem = cw_smem_host(Q);
        if (Q.cw_smem <= 110 * 1024) { P = Q; P.cw = 1; break; }
      }
    }
    if ((W + 3 * H) * 4 > kSmemBudget) return fail(BBX_SPEC_MISMATCH, "output too large for the device plan");
  }
  if (P.value_mode == VAL_LUT) {   // exact u8 -> output table (pipeline.py:158-160 arithmetic)
    const int osz = dtype_size(out_dt);
    std::vector<uint8_t> lut((size_t)C * 256 * osz);
    for (int k = 0; k < C; ++k)
      for (int v = 0; v < 256; ++v) {
        float x = (float)v;
        for (int i = 0; i < P.n_vops; ++i) {
          volatile float t = x - P.vop_mean[i][k];
          x = t / P.vop_std[i][k];
        }
        uint8_t* at = &lut[((size_t)k * 256 + v) * osz];
        if (out_dt == BBX_F32) std::memcpy(at, &x, 4);
        else { uint16_t b = out_dt == BBX_F16 ? f32_to_f16_bits(x) : f32_to_bf16_bits(x); std::memcpy(at, &b, 2); }
      }
    CK(cudaMalloc(&pl.d_lut, lut.size()));
    CK(cudaMemcpy(pl.d_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice));
    if (P.cw && (out_dt == BBX_F16 || out_dt == BBX_BF16) && prove_affine(P, C, lut, out_dt)) {
      P.cw_affine = 1;
      P.cw_smem = cw_smem_host(P);   // no value table in shared memory
    }
  }
  // one pass over the row table: exact staging capacity, RLE presence
  int64_t mx = 0;
  bool rle = false, jpeg = false;
  if (f.info.kind == 4) {
    for (int64_t i = 0; i < ds->num_samples; ++i) {
      ImageCell c = image_cell(ds, i, f);
      mx = std::max<int64_t>(mx, (int64_t)c.length);
      rle |= c.codec == CODEC_RLE;
      jpeg |= c.codec == CODEC_JPEG;
    }
  } else {
    mx = f.array_nbytes;
  }
  pl.max_payload = mx;
  pl.field_has_rle = rle;
  pl.field_has_jpeg = jpeg;
  if (jpeg) {   // bounds over every header a cell of this field can carry (dims checked per sample)
    const int64_t mh = f.info.max_height, mw = f.info.max_width;
    pl.jpeg_blocks_cap = (int64_t)f.info.channels * (2 * ((mh + 15) / 16)) * (2 * ((mw + 15) / 16));
    pl.jpeg_int_cap = ((mh + 7) / 8) * ((mw + 7) / 8);
  }
  return BBX_OK;
}

// Host-side per-sample work for one plan: descriptor + RNG params + checks.
// Returns false (and fills err) when the sample must be skipped.
// Host twins of the kernel's back_x/back_y (image_kernel.cuh): the composed
// remaps are monotone, so the referenced canvas range is spanned by the ends.
static int host_back_y(const PlanDev& P, const int32_t* prm, int y) {
  for (int i = P.n_remaps - 1; i >= 0; --i) {
    const Remap& m = P.remaps[i];
    if (m.kind == BBX_OP_CROP) y += prm[m.prm];
    else if (m.kind == BBX_OP_RESIZE) y = (int)(((int64_t)y * m.in_h) / m.out_h);
  }
  return y;
}
static int host_back_x(const PlanDev& P, const int32_t* prm, int x) {
  for (int i = P.n_remaps - 1; i >= 0; --i) {
    const Remap& m = P.remaps[i];
    if (m.kind == BBX_OP_CROP) x += prm[m.prm + 1];
    else if (m.kind == BBX_OP_FLIP) { if (prm[m.prm]) x = m.in_w - 1 - x; }
    else if (m.kind == BBX_OP_RESIZE) x = (int)(((int64_t)x * m.in_w) / m.out_w);
  }
  return x;
}
// Image rows [y0, y1) x columns [x0, x1) a RAW sample's chain reads (empty when
// the output only sees zero padding).  Resample decoders read exactly their
// window (lin_axis indices stay inside it).
static void read_window(const PlanDev& P, const SampleDesc* d, const int32_t* prm, int* y0, int* y1, int* x0, int* x1) {
  if (P.src_kind == SRC_RESAMPLE) {
    *y0 = prm[0]; *y1 = prm[0] + prm[2]; *x0 = prm[1]; *x1 = prm[1] + prm[3];
    return;
  }
  int ya = host_back_y(P, prm, 0), yb = host_back_y(P, prm, P.out_h - 1);
  int xa = host_back_x(P, prm, 0), xb = host_back_x(P, prm, P.out_w - 1);
  *y0 = std::min(ya, yb); *y1 = std::min(std::max(ya, yb) + 1, (int)d->h);
  *x0 = std::min(xa, xb); *x1 = std::min(std::max(xa, xb) + 1, (int)d->w);
  if (*y0 >= *y1 || *x0 >= *x1) { *y0 = *y1 = *x0 = *x1 = 0; }
}

static bool fill_desc(const bbx_dataset* ds, const Plan& pl, int64_t i, uint64_t seed, uint64_t epoch, uint8_t* desc,
                      uint64_t* src_off, uint32_t* len, HostErr& err, int64_t pos, int plan_idx) {
  const Field& f = ds->fields[pl.field_index];
  SampleDesc* d = reinterpret_cast<SampleDesc*>(desc);
  int32_t* prm = reinterpret_cast<int32_t*>(desc + kDescHeader);
  std::memset(desc, 0, pl.dev.desc_stride);
  d->index_lo = (int32_t)i;
  auto bad = [&](int code, const char* fmt, auto... args) {
    d->skip = 1;
    if (err.pos < 0 || pos < err.pos || (pos == err.pos && plan_idx < err.plan)) {
      char buf[512];
      std::snprintf(buf, sizeof buf, fmt, args...);
      err.pos = pos; err.plan = plan_idx; err.code = code; err.msg = buf;
    }
    return false;
  };
  if (f.info.kind == 4) {
    ImageCell c = image_cell(ds, i, f);
    d->h = (uint16_t)c.h; d->w = (uint16_t)c.w; d->c = (uint8_t)c.c; d->codec = (uint8_t)c.codec;
    *src_off = c.offset; *len = (uint32_t)c.length;
    d->len = (uint32_t)c.length;
    if (c.length > 0xFFFFFFFFull) return bad(BBX_CORRUPT_PAYLOAD, "payload of %llu bytes is too large", (unsigned long long)c.length);
    // the payload must lie inside the heap: staging reads the mmap and resident /
    // paged plans read the HBM heap image, both of which span exactly the heap
    if (c.length && ((int64_t)c.offset < ds->heap_offset || c.offset + c.length > (uint64_t)ds->alloc_table_offset))
      return bad(BBX_CORRUPT_PAYLOAD, "payload [%llu, %llu) lies outside the heap [%lld, %lld)",
                 (unsigned long long)c.offset, (unsigned long long)(c.offset + c.length), (long long)ds->heap_offset,
                 (long long)ds->alloc_table_offset);
    int mh = f.info.max_height, mw = f.info.max_width, ch = f.info.channels;
    if (pl.dev.src_kind == SRC_DECODE) {        // decode_image(out[:h, :w, :]) shape check
      if (c.h > mh || c.w > mw || c.c != ch)
        return bad(BBX_SCHEMA_MISMATCH, "output buffer must be u8 (%d, %d, %d), got uint8 (%d, %d, %d)", c.h, c.w, c.c,
                   std::min(c.h, mh), std::min(c.w, mw), ch);
    } else if (c.h > mh || c.w > mw || c.c != ch) {
      return bad(BBX_SCHEMA_MISMATCH, "image %dx%dx%d does not fit field (%d, %d, %d)", c.h, c.w, c.c, mh, mw, ch);
    }
    int64_t n = (int64_t)c.h * c.w * c.c;
    if (c.codec == CODEC_RAW) {
      if ((int64_t)c.length != n) return bad(BBX_CORRUPT_PAYLOAD, "raw payload is %lld bytes, expected %lld",
                                             (long long)c.length, (long long)n);
    } else if (c.codec == CODEC_RLE) {
      if (c.length % 5) return bad(BBX_CORRUPT_PAYLOAD, "rle payload length is not a multiple of 5");
    } else if (c.codec == CODEC_SUB2) {
      int64_t m = (int64_t)((c.h + 1) / 2) * ((c.w + 1) / 2) * c.c;
      if ((int64_t)c.length != m) return bad(BBX_CORRUPT_PAYLOAD, "subsampled payload is %lld bytes, expected %lld",
                                             (long long)c.length, (long long)m);
    } else if (c.codec == CODEC_JPEG) {
      if (c.length < 4) return bad(BBX_CORRUPT_PAYLOAD, "jpeg: missing SOI marker");
      if (!pl.field_has_jpeg) return bad(BBX_CORRUPT_PAYLOAD, "jpeg sample in a field compiled without JPEG");
    } else {
      return bad(BBX_CORRUPT_PAYLOAD, "unknown codec %d", c.codec);
    }
    if (n == 0) return bad(BBX_SCHEMA_MISMATCH, "image dims must all be >= 1");
  } else {
    *src_off = u64_cell(ds, i, f);
    *len = (uint32_t)f.array_nbytes;
    d->len = (uint32_t)f.array_nbytes;
    if ((int64_t)*src_off < ds->heap_offset || *src_off + f.array_nbytes > (uint64_t)ds->alloc_table_offset)
      return bad(BBX_CORRUPT_PAYLOAD, "array payload [%llu, %llu) lies outside the heap [%lld, %lld)",
                 (unsigned long long)*src_off, (unsigned long long)(*src_off + f.array_nbytes),
                 (long long)ds->heap_offset, (long long)ds->alloc_table_offset);
  }
  // per-sample stream (loader.py:339): stream_seed(seed, TAG_SAMPLE, epoch, i, fidx)
  Rng r(fold(fold(fold(fold(seed, 2), epoch), (uint64_t)i), (uint64_t)pl.field_index));
  for (const Draw& dr : pl.draws) {
    switch (dr.kind) {
      case BBX_OP_RRC: {
        int t, l, hh, ww;
        rrc_window(r, d->h, d->w, dr.scale, dr.ratio, &t, &l, &hh, &ww, dr.log_ratio);
        prm[0] = t; prm[1] = l; prm[2] = hh; prm[3] = ww;
        break;
      }
      case BBX_OP_CENTERCROP: {
        int t, l, hh, ww;
        center_window(d->h, d->w, dr.p, &t, &l, &hh, &ww);
        prm[0] = t; prm[1] = l; prm[2] = hh; prm[3] = ww;
        break;
      }
      case BBX_OP_CROP:                          // pipeline.py:199-202: top, then left
        prm[dr.slot] = (int32_t)r.below((uint64_t)(dr.in_h - dr.h + 1));
        prm[dr.slot + 1] = (int32_t)r.below((uint64_t)(dr.in_w - dr.w + 1));
        break;
      case BBX_OP_FLIP:                          // pipeline.py:177-181
        prm[dr.slot] = r.chance(dr.p) ? 1 : 0;
        break;
    }
  }
  return true;
}

static void pipeline_loop(bbx_loader* L);

// Table pool ids for one JPEG header (registering unseen tables).  Callers hold T.mu.
static uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h = 1469598103934665603ull) {
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}
// Table keys and hashes are built outside the registry lock; the lock covers
// only the lookup (and, for a table never seen before, its registration).
struct HuffKey { uint8_t key[1 + 16 + 256]; size_t n; uint64_t hv; };
static void huff_key(const JpegHeader::Huff& h, bool is_ac, HuffKey* k) {
  k->key[0] = is_ac ? 'A' : 'D';
  std::memcpy(k->key + 1, h.counts, 16);
  std::memcpy(k->key + 17, h.vals, h.nvals);
  k->n = 17 + h.nvals;
  k->hv = fnv1a(k->key, k->n);
}
static int jpeg_table_id(JpegTables& T, const JpegHeader::Huff& h, bool is_ac, const HuffKey& k, int* id) {
  for (auto [it, end] = T.hmap.equal_range(k.hv); it != end; ++it) {
    const auto& e = T.hkey[it->second];
    if (e.size() == k.n && !std::memcmp(e.data(), k.key, k.n)) { *id = it->second; return 0; }
  }
  if (T.n_huff >= kJpegMaxHuff) return 2;
  if (!jpeg_build_huff(h, is_ac, &T.h_huff[T.n_huff])) return 1;
  T.hkey.emplace_back(k.key, k.key + k.n);
  T.hmap.emplace(k.hv, T.n_huff);
  *id = T.n_huff++;
  return 0;
}
static int jpeg_quant_id(JpegTables& T, const JpegHeader::Quant& q, uint64_t hv, int* id) {
  const uint8_t* key = reinterpret_cast<const uint8_t*>(q.q);
  for (auto [it, end] = T.qmap.equal_range(hv); it != end; ++it)
    if (!std::memcmp(T.qkey[it->second].data(), key, sizeof q.q)) { *id = it->second; return 0; }
  if (T.n_quant >= kJpegMaxQuant) return 2;
  std::memcpy(T.h_quant[T.n_quant].q, q.q, sizeof q.q);
  T.qkey.emplace_back(key, key + sizeof q.q);
  T.qmap.emplace(hv, T.n_quant);
  *id = T.n_quant++;
  return 0;
}

// Host half of the JPEG decode of one sample: parse the header, check it
// against the cell, resolve table ids and size the device work.
static bool jpeg_prepare(bbx_loader* L, const Plan& pl, const uint8_t* pay, uint32_t len, SampleDesc* d, JpegDesc* J,
                         std::vector<uint32_t>* starts, HostErr& err, int64_t pos, int plan_idx) {
  auto bad = [&](const char* m) {
    d->skip = 1;
    if (err.pos < 0 || pos < err.pos || (pos == err.pos && plan_idx < err.plan)) {
      err.pos = pos; err.plan = plan_idx; err.code = BBX_CORRUPT_PAYLOAD; err.msg = m;
    }
    return false;
  };
  JpegHeader H;
  char msg[256];
  if (jpeg_parse_header(pay, len, &H, msg, sizeof msg)) return bad(msg);
  if (H.height != d->h || H.width != d->w || H.ncomp != d->c) {
    std::snprintf(msg, sizeof msg, "jpeg: header says %dx%dx%d, cell says %dx%dx%d", H.height, H.width, H.ncomp,
                  d->h, d->w, d->c);
    return bad(msg);
  }
  std::memset(J, 0, sizeof *J);
  int hmax = 1, vmax = 1;
  for (int i = 0; i < H.ncomp; ++i) { hmax = std::max(hmax, H.comp[i].h); vmax = std::max(vmax, H.comp[i].v); }
  const int mx = H.ncomp == 1 ? (H.width + 7) / 8 : (H.width + 8 * hmax - 1) / (8 * hmax);
  const int my = H.ncomp == 1 ? (H.height + 7) / 8 : (H.height + 8 * vmax - 1) / (8 * vmax);
  uint32_t blocks = 0;
  int mcu_off = 0;
  JpegTables& T = L->jt;
  HuffKey kd[3], ka[3];
  uint64_t kq[3];
  for (int i = 0; i < H.ncomp; ++i) {
    const auto& c = H.comp[i];
    huff_key(H.dc[c.td], false, &kd[i]);
    huff_key(H.ac[c.ta], true, &ka[i]);
    kq[i] = fnv1a(reinterpret_cast<const uint8_t*>(H.qt[c.tq].q), sizeof H.qt[c.tq].q);
  }
  int ids[3][3];
  {
    std::lock_guard<std::mutex> g(T.mu);
    for (int i = 0; i < H.ncomp; ++i) {
      const auto& c = H.comp[i];
      int r;
      if ((r = jpeg_table_id(T, H.dc[c.td], false, kd[i], &ids[i][0])) ||
          (r = jpeg_table_id(T, H.ac[c.ta], true, ka[i], &ids[i][1])) || (r = jpeg_quant_id(T, H.qt[c.tq], kq[i], &ids[i][2])))
        return bad(r == 2 ? "jpeg: too many distinct tables for the device table pool" : "jpeg: bad Huffman table");
    }
  }
  for (int i = 0; i < H.ncomp; ++i) {
    const auto& c = H.comp[i];
    JComp& o = J->comp[i];
    const int dc = ids[i][0], ac = ids[i][1], q = ids[i][2];
    o.dc = (uint16_t)dc; o.ac = (uint16_t)ac; o.q = (uint16_t)q;
    o.h = (uint8_t)c.h; o.v = (uint8_t)c.v;
    o.bw = (uint16_t)(H.ncomp == 1 ? mx : mx * c.h);
    o.bh = (uint16_t)(H.ncomp == 1 ? my : my * c.v);
    o.dw = (uint16_t)(((int64_t)H.width * c.h + hmax - 1) / hmax);
    o.dh = (uint16_t)(((int64_t)H.height * c.v + vmax - 1) / vmax);
    o.blk_off = (uint32_t)mcu_off;
    mcu_off += H.ncomp == 1 ? 1 : c.h * c.v;
    J->plane_blk[i] = blocks;
    blocks += (uint32_t)o.bw * o.bh;
  }
  const uint32_t total = (uint32_t)mx * my;
  J->scan_off = H.scan_off;
  // the scan data ends at the EOI marker (last 0xFFD9; inside coded data 0xFF
  // is always followed by 0x00); a file without one is decoded as truncated
  uint32_t end = len;
  for (int64_t q = (int64_t)len - 2; q >= (int64_t)H.scan_off; --q)
    if (pay[q] == 0xFF && pay[q + 1] == 0xD9) { end = (uint32_t)q; break; }
  J->scan_end = end;
  J->mcus_x = (uint16_t)mx; J->mcus_y = (uint16_t)my;
  J->restart = H.restart ? (uint32_t)H.restart : total;
  J->n_int = (total + J->restart - 1) / J->restart;
  J->ncomp = (uint8_t)H.ncomp; J->hmax = (uint8_t)hmax; J->vmax = (uint8_t)vmax;
  J->n_blocks = blocks;
  int bpm = 0;                                   // MCU block order (T.81 A.2.3): comps, then rows, then columns
  for (int i = 0; i < H.ncomp; ++i)
    for (int v = 0; v < J->comp[i].v; ++v)
      for (int h = 0; h < J->comp[i].h; ++h, ++bpm)
        J->sched |= (uint64_t)(i | v << 2 | h << 3) << (4 * bpm);
  J->bpm = (uint8_t)bpm;
  if ((int64_t)blocks > pl.jpeg_blocks_cap || (int64_t)J->n_int > pl.jpeg_int_cap)
    return bad("jpeg: geometry exceeds the field's device capacity");
  // Restart intervals (T.81 B.2.5): the entropy-coded bytes between RSTn
  // markers.  A marker is 0xFF followed by neither 0x00 (stuffing) nor 0xFF
  // (fill); every one inside the scan must be the next RSTn in sequence, and
  // there must be exactly n_int - 1 of them.  starts[k] = interval k's first byte.
  starts->clear();
  starts->reserve(J->n_int);
  starts->push_back(H.scan_off);
  char m2[96];
  for (uint32_t q = H.scan_off; q + 1 < end;) {
    const void* f = std::memchr(pay + q, 0xFF, end - 1 - q);
    if (!f) break;
    q = (uint32_t)(static_cast<const uint8_t*>(f) - pay);
    const uint8_t c = pay[q + 1];
    if (c == 0x00) { q += 2; continue; }
    if (c == 0xFF) { q += 1; continue; }
    if ((c & 0xF8) != 0xD0) {
      std::snprintf(m2, sizeof m2, "jpeg: restart marker count %d does not match the header", -1);
      return bad(m2);
    }
    const uint32_t n = (uint32_t)starts->size();   // this is RST number n - 1 of the scan
    if (n >= J->n_int) {
      std::snprintf(m2, sizeof m2, "jpeg: restart marker count %u does not match the header", n);
      return bad(m2);
    }
    if ((uint32_t)(c & 7) != ((n - 1) & 7u)) return bad("jpeg: restart markers out of sequence");
    starts->push_back(q + 2);
    q += 2;
  }
  if (starts->size() != J->n_int) {
    std::snprintf(m2, sizeof m2, "jpeg: restart marker count %u does not match the header", (uint32_t)starts->size() - 1);
    return bad(m2);
  }
  return true;
}

// staged per JPEG plan: JpegDesc[B] | u32 interval prefix[B+1] | u64 block prefix[B+1]
static size_t jpeg_iprefix_off(int B) { return (size_t)B * sizeof(JpegDesc); }
static size_t jpeg_bprefix_off(int B) { return (jpeg_iprefix_off(B) + (size_t)(B + 1) * 4 + 7) / 8 * 8; }
static size_t jpeg_block_bytes(int B) { return jpeg_bprefix_off(B) + (size_t)(B + 1) * 8; }



static int finalize_impl(bbx_loader* L);
// Pinned staging memory is allocated (and first touched) with the calling
// thread bound to the GPU's NUMA node, so the pages sit next to the GPU's PCIe
// root: the gather writes them and the DMA reads them without crossing sockets.
static int finalize(bbx_loader* L) {
  if (L->finalized || L->local_cpus.empty()) return finalize_impl(L);
  cpu_set_t old;
  const bool have_old = pthread_getaffinity_np(pthread_self(), sizeof old, &old) == 0;
  set_affinity(pthread_self(), L->local_cpus);
  const int r = finalize_impl(L);
  if (have_old) pthread_setaffinity_np(pthread_self(), sizeof old, &old);
  return r;
}
static int finalize_impl(bbx_loader* L) {
  if (L->finalized) return BBX_OK;
  CK(cudaSetDevice(L->device));
  // slot layout: [idx: B*8][desc blocks per plan][one compact payload region]
  size_t off = 0;
  L->idx_off = 0;
  off += (size_t)L->batch * 8;
  off = (off + 255) / 256 * 256;
  L->desc_off.assign(L->plans.size(), 0);
  for (size_t p = 0; p < L->plans.size(); ++p) {
    if (L->plans[p].scalar) continue;
    L->desc_off[p] = off;
    off += (size_t)L->batch * L->plans[p].dev.desc_stride;
    off = (off + 255) / 256 * 256;
  }
  L->jpeg_off.assign(L->plans.size(), 0);
  bool any_jpeg = false;
  for (size_t p = 0; p < L->plans.size(); ++p) {
    if (L->plans[p].scalar || !L->plans[p].field_has_jpeg) continue;
    any_jpeg = true;
    L->jpeg_off[p] = off;
    off += jpeg_block_bytes(L->batch) + (size_t)L->batch * L->plans[p].jpeg_int_cap * 4;   // + interval starts
    off = (off + 255) / 256 * 256;
  }
  L->desc_bytes = off;
  bool codec_stage = false;           // RLE / JPEG payloads are expanded from a staged copy
  for (const auto& pl : L->plans) codec_stage |= !pl.scalar && (pl.field_has_rle || pl.field_has_jpeg);
  // zero-copy gather: the pinned heap's window rows are gathered into the slot by a
  // kernel (PCIe reads, one host DRAM read per byte), and K1 reads them from HBM as a
  // staged batch; direct zero-copy (K1 pulling its rows over PCIe itself) keeps too few
  // reads in flight.  Not for RLE / JPEG plans: their decode kernels fill the SMs, so a
  // gather kernel would serialise with them where the copy engine's DMA overlaps them
  // (configs[2]: 1.03 vs 1.47 M img/s)
  const bool zc_ok = !L->ds->d_heap && L->zero_copy && L->ds->h_heap_dev && !codec_stage;
  L->zcg = zc_ok && L->zc_gather && !L->direct_io && L->pp.capacity == 0;
  L->zc = zc_ok && !L->zcg;
  if (L->zcg) {
    size_t np = 0;
    for (const auto& pl : L->plans) np += pl.scalar ? 0 : 1;
    L->gcopy_off = off;
    off += (size_t)L->batch * np * sizeof(GatherCopy);
    off = (off + 255) / 256 * 256;
    L->desc_bytes = off;
  }
  L->payload_dev = L->ds->d_heap ? L->ds->d_heap : (L->zc ? L->ds->h_heap_dev : nullptr);
  bool resident = L->payload_dev != nullptr;
  L->pay_base = off;
  for (size_t p = 0; p < L->plans.size(); ++p) {   // capacity: every sample's whole payload
    if (L->plans[p].scalar || resident) continue;
    off += (size_t)L->batch * (size_t)((L->plans[p].max_payload + 15) / 16 * 16);
  }
  L->slot_bytes = off + 256;
  size_t nplans = L->plans.size();
  for (auto& S : L->slots) {
    CK(cudaHostAlloc(&S.h_stage, L->slot_bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&S.d_stage, L->slot_bytes));
    S.cap = L->slot_bytes;
    CK(cudaMalloc(&S.d_status, sizeof(SampleStatus) * L->batch * std::max<size_t>(nplans, 1)));
    CK(cudaHostAlloc(&S.h_status, sizeof(SampleStatus) * L->batch * std::max<size_t>(nplans, 1), cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&S.h2d_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S.release, cudaEventDisableTiming));
    CK(cudaEventCreate(&S.k0));
    CK(cudaEventCreate(&S.k1));
  }
  for (auto& pl : L->plans) {
    if (pl.scalar || !pl.dev.cw) continue;
    for (int k = 0; k < kStreams; ++k) {
      CK(cudaMalloc(&pl.d_ticket[k], 16));
      CK(cudaMemset(pl.d_ticket[k], 0, 16));
    }
  }
  for (auto& pl : L->plans) {
    if (pl.scalar || pl.dev.src_kind == SRC_ARRAY) continue;
    pl.d_tables.assign(L->nslots, nullptr);
    for (int s = 0; s < L->nslots; ++s) CK(cudaMalloc(&pl.d_tables[s], (size_t)L->batch * pl.dev.tab_stride * 4 + 64));
  }
  for (auto& pl : L->plans) {
    if (pl.scalar || !(pl.field_has_rle || pl.field_has_jpeg)) continue;
    pl.d_scratch.assign(L->nslots, nullptr);
    for (int s = 0; s < L->nslots; ++s) CK(cudaMalloc(&pl.d_scratch[s], (size_t)L->batch * pl.dev.scratch_bytes + 64));
  }
  for (auto& pl : L->plans) {
    if (pl.scalar || !pl.field_has_jpeg) continue;
    if (L->jpeg_cache) {
      pl.jcache.resize(L->ds->num_samples);
      pl.jstarts.assign(L->ds->num_samples, {});
      pl.jcached.assign(L->ds->num_samples, 0);
    }
    const size_t blocks = (size_t)L->batch * pl.jpeg_blocks_cap, ints = (size_t)L->batch * pl.jpeg_int_cap;
    for (int k = 0; k < kStreams; ++k) {
      CK(cudaMalloc(&pl.d_coef[k], blocks * 128 + 256));
      CK(cudaMalloc(&pl.d_planes[k], blocks * 64 + 256));
    }
  }
  if (any_jpeg && !L->jt.d_huff) {
    JpegTables& T = L->jt;
    CK(cudaHostAlloc(&T.h_huff, sizeof(JHuff) * kJpegMaxHuff, cudaHostAllocDefault));
    CK(cudaHostAlloc(&T.h_quant, sizeof(JQuant) * kJpegMaxQuant, cudaHostAllocDefault));
    CK(cudaMalloc(&T.d_huff, sizeof(JHuff) * kJpegMaxHuff));
    CK(cudaMalloc(&T.d_quant, sizeof(JQuant) * kJpegMaxQuant));
  }
  // Every sample's JPEG header, parsed once up front on the pool when the file
  // sits comfortably in RAM (reading the headers touches every sample): the
  // first epoch's batches then cost what later ones do.  Samples whose header
  // does not parse stay uncached and report their error in their batch.
  // A distributed loader names the samples it will see first (its shard of the
  // first epoch, bbx_loader_prefetch_headers), so ranks do not all parse every header.
  if (any_jpeg && L->jpeg_cache && L->jpeg_prefetch) {
    const bbx_dataset* ds = L->ds;
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    if ((double)ds->map_len < 0.25 * (double)pages * (double)psz) {
      const bool subset = !L->prefetch_set.empty();
      const int64_t n = subset ? (int64_t)L->prefetch_set.size() : ds->num_samples;
      for (auto& pl : L->plans) {
        if (pl.scalar || !pl.field_has_jpeg) continue;
        const Field& f = ds->fields[pl.field_index];
        L->pool->parallel_for(n, [&](int64_t k) {
          const int64_t i = subset ? L->prefetch_set[k] : k;
          if (i < 0 || i >= ds->num_samples || pl.jcached[i]) return;
          const ImageCell c = image_cell(ds, i, f);
          if (c.codec != CODEC_JPEG || c.length > 0xFFFFFFFFull || (int64_t)c.offset < ds->heap_offset ||
              c.offset + c.length > (uint64_t)ds->alloc_table_offset)
            return;
          SampleDesc d{};
          d.h = (uint16_t)c.h; d.w = (uint16_t)c.w; d.c = (uint8_t)c.c;
          JpegDesc J;
          HostErr e;
          if (jpeg_prepare(L, pl, ds->map + c.offset, (uint32_t)c.length, &d, &J, &pl.jstarts[i], e, 0, 0)) {
            pl.jcache[i] = J;
            pl.jcached[i] = 1;
          }
        });
      }
    }
  }
  // Staged loaders read payloads from the mmap: populate its page tables once,
  // in parallel on the staging threads, when the file comfortably fits in RAM
  // (MADV_POPULATE_READ), so batches do not pay a minor fault per 4 KiB page on
  // the first touch of every sample (the OS page cache keeps the data; only the
  // process's mapping is filled in).  Once per dataset.
  if (!resident && !L->direct_io) {
    bbx_dataset* ds = L->ds;
    std::lock_guard<std::mutex> g(ds->reg_mu);
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    if (!ds->populated && (double)ds->map_len < 0.25 * (double)pages * (double)psz) {
      const int64_t chunk = 64ll << 20, n = ((int64_t)ds->map_len + chunk - 1) / chunk;
      L->pool->parallel_for(n, [&](int64_t c) {
        const int64_t a = c * chunk, m = std::min<int64_t>(chunk, (int64_t)ds->map_len - a);
#ifndef MADV_POPULATE_READ
#define MADV_POPULATE_READ 22
#endif
        if (madvise((void*)(ds->map + a), (size_t)m, MADV_POPULATE_READ) != 0) {   // older kernels: touch
          volatile uint8_t sink = 0;
          for (int64_t q = 0; q < m; q += psz) sink ^= ds->map[a + q];
        }
      });
      ds->populated = true;
    }
  }
  L->th = std::thread(pipeline_loop, L);
  set_affinity(L->th.native_handle(), L->local_cpus);
  L->finalized = true;
  return BBX_OK;
}

// The per-batch pipeline body (runs on the loader thread).
// Window rows into the pinned slot: 16-byte-aligned destination rows written
// with non-temporal stores (no read-for-ownership of the slot: the gather is
// host-memory bound, and the slot is next read by the H2D DMA, not the CPU).
// A row's last chunk may read up to 15 bytes past it (never past the mapping).
static void gather_rows(uint8_t* dst, uint32_t dst_stride, const uint8_t* src, uint32_t src_stride, uint32_t row_bytes,
                        uint32_t rows, const uint8_t* src_end) {
#if defined(__SSE2__)
  const uint32_t n16 = (row_bytes + 15) / 16;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint8_t* s = src + (size_t)r * src_stride;
    uint8_t* d = dst + (size_t)r * dst_stride;
    if (s + (size_t)n16 * 16 > src_end || (reinterpret_cast<uintptr_t>(d) & 15)) { std::memcpy(d, s, row_bytes); continue; }
    for (uint32_t i = 0; i < n16; ++i)
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16 * i), _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16 * i)));
  }
  _mm_sfence();   // the streaming stores are visible before the pool reports the batch gathered
#else
  for (uint32_t r = 0; r < rows; ++r) std::memcpy(dst + (size_t)r * dst_stride, src + (size_t)r * src_stride, row_bytes);
  (void)src_end;
#endif
}

// ------------------------------------------------------------------ page pool
// Distinct heap pages of sample i, ascending (reader.py:414-424 sample_pages).
// Pages outside the heap are left out (the sample fails at its descriptor).
static void sample_pages(const bbx_dataset* ds, int64_t i, std::vector<int64_t>& out) {
  out.clear();
  const int64_t ps = ds->page_size, np = (ds->alloc_table_offset - ds->heap_offset) / ps;
  auto add = [&](uint64_t off, uint64_t len) {
    if (!len) return;
    const int64_t a = ((int64_t)off - ds->heap_offset) / ps, b = ((int64_t)(off + len - 1) - ds->heap_offset) / ps;
    for (int64_t q = std::max<int64_t>(a, 0); q <= std::min<int64_t>(b, np - 1); ++q) out.push_back(q);
  };
  for (const Field& f : ds->fields) {
    const uint8_t* c = ds->rows + i * ds->row_width + f.info.cell_offset;
    uint64_t off, len;
    if (f.info.kind == 2) { std::memcpy(&off, c, 8); add(off, (uint64_t)f.array_nbytes); }
    else if (f.info.kind == 3 || f.info.kind == 4) { std::memcpy(&off, c, 8); std::memcpy(&len, c + 8, 8); add(off, len); }
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

// The epoch's page plan: the trace loader.py:276-291 builds (each batch's
// samples' pages, in batch order), the CapacityTooSmall check of loader.py:
// 286-289, and the farthest-next-use schedule of reader.py:112-141 (victim =
// the resident page with the largest (next use, page)); fetch / reload counts
// are the schedule's planned ones.
static int plan_epoch(bbx_loader* L, const int64_t* idx, const int32_t* blen, int32_t nb, PagePlan& P) {
  const bbx_dataset* ds = L->ds;
  const int64_t K = L->pp.capacity, np = (ds->alloc_table_offset - ds->heap_offset) / ds->page_size;
  std::vector<int64_t> pg, stamp((size_t)np, -1);
  P.batch_off.assign(1, 0);
  int64_t k = 0;
  for (int32_t b = 0; b < nb; ++b) {
    int64_t distinct = 0;
    for (int32_t j = 0; j < blen[b]; ++j, ++k) {
      const int64_t i = idx[k];
      P.idx.push_back(i);
      P.trace_off.push_back((int64_t)P.trace.size());
      if (i >= 0 && i < ds->num_samples) sample_pages(ds, i, pg); else pg.clear();
      for (int64_t q : pg) {
        P.trace.push_back(PageStep{q, -1, 0, 0, 0});
        if (stamp[q] != b) { stamp[q] = b; ++distinct; }
      }
    }
    if (distinct > K)
      return fail(BBX_CAPACITY_TOO_SMALL, "batch touches %lld pages, cache holds %lld", (long long)distinct,
                  (long long)K);
    P.batch_off.push_back(k);
  }
  P.trace_off.push_back((int64_t)P.trace.size());
  const int64_t T = (int64_t)P.trace.size(), INF = T + 1;
  std::vector<int64_t> next_use((size_t)T), last_seen((size_t)np, INF);
  for (int64_t t = T - 1; t >= 0; --t) {
    next_use[t] = last_seen[P.trace[t].page];
    last_seen[P.trace[t].page] = t;
  }
  std::set<std::pair<int64_t, int64_t>> res;        // (next use, page) of the resident pages
  std::vector<int64_t> cur((size_t)np, -1), last_pos((size_t)np, -1);
  std::vector<uint8_t> seen((size_t)np, 0);
  P.phys_needed = K;
  for (int32_t b = 0; b < nb; ++b) {
    const int64_t t0 = P.trace_off[P.batch_off[b]], t1 = P.trace_off[P.batch_off[b + 1]];
    int64_t deferred = 0;
    for (int64_t t = t0; t < t1; ++t) {
      PageStep& st = P.trace[t];
      const int64_t q = st.page;
      if (cur[q] >= 0) {
        res.erase({cur[q], q});
      } else {
        if ((int64_t)res.size() >= K) {
          auto it = std::prev(res.end());
          const int64_t v = it->second;
          res.erase(it);
          cur[v] = -1;
          st.victim = v;
          st.deferred = last_pos[v] >= t0 ? 1 : 0;   // read by this batch's kernels: recycle after them
          deferred += st.deferred;
        }
        st.fetch = 1;
        st.reload = seen[q];
        seen[q] = 1;
        ++P.fetches;
        P.reloads += st.reload;
      }
      cur[q] = next_use[t];
      res.insert({cur[q], q});
      last_pos[q] = t;
    }
    P.phys_needed = std::max(P.phys_needed, K + deferred);
  }
  return BBX_OK;
}

// Fetch heap page `page` into physical pool slot `ph`: once the last batch that
// read the slot is done, the page's bytes go mmap -> pinned page buffer (the
// staging pool's threads) -> H2D on the copy stream (reader.py:379-384 _fetch_page,
// with the strategy's fetch latency spun before it as in reader.py:247-248).
static int fetch_page(bbx_loader* L, int64_t page, int64_t ph) {
  PagePool& PP = L->pp;
  const bbx_dataset* ds = L->ds;
  if (PP.user_ring[ph] >= 0 && L->slots[PP.user_ring[ph]].serial == PP.user_serial[ph])
    CK(cudaStreamWaitEvent(L->copy_st, L->slots[PP.user_ring[ph]].done, 0));
  const int k = PP.buf_next;
  PP.buf_next = (k + 1) % kPageBufs;
  if (PP.buf_used[k]) CK(cudaEventSynchronize(PP.buf_ev[k]));
  if (PP.fetch_latency_s > 0) {
    const auto until = std::chrono::steady_clock::now() + std::chrono::duration<double>(PP.fetch_latency_s);
    while (std::chrono::steady_clock::now() < until) {}
  }
  const int64_t ps = ds->page_size, off = ds->heap_offset + page * ps;
  const int64_t len = std::min<int64_t>(ps, ds->alloc_table_offset - off);
  uint8_t* dst = PP.h_buf + (size_t)k * ps;
  const int64_t chunk = 1 << 20, n = (len + chunk - 1) / chunk;
  L->pool->parallel_for(n, [&](int64_t c) {
    const int64_t a = c * chunk, m = std::min(chunk, len - a);
    std::memcpy(dst + a, ds->map + off + a, (size_t)m);
  });
  CK(cudaMemcpyAsync(PP.d_pool + (size_t)ph * ps, dst, (size_t)len, cudaMemcpyHostToDevice, L->copy_st));
  CK(cudaEventRecord(PP.buf_ev[k], L->copy_st));
  PP.buf_used[k] = true;
  std::lock_guard<std::mutex> g(L->stats_mu);
  L->stats.page_fetches += 1;
  L->stats.h2d_bytes += len;
  return BBX_OK;
}

// This batch's part of the installed plan: its fetches / evictions in trace
// order, and the pool address of every sample payload that lies in one page
// (addr[p][pos]; null: staged like an OsCache payload -- oversized blobs).
static int page_batch(bbx_loader* L, Slot& S, int count, std::vector<std::vector<const uint8_t*>>& addr,
                      std::vector<int64_t>& read_slots, std::vector<int64_t>& deferred) {
  PagePool& PP = L->pp;
  const bbx_dataset* ds = L->ds;
  PagePlan* Pp;
  {
    std::lock_guard<std::mutex> g(L->mu);
    if (PP.plans.empty()) return fail(BBX_INVALID_ARGUMENT, "page pool: batch submitted without an epoch plan");
    Pp = &PP.plans.front();
  }
  PagePlan& P = *Pp;
  const int32_t b = P.next;
  const int64_t k0 = P.batch_off[b], k1 = P.batch_off[b + 1];
  if (k1 - k0 != count || std::memcmp(&P.idx[k0], S.idx.data(), (size_t)count * 8))
    return fail(BBX_INVALID_ARGUMENT, "page pool: batch does not follow the installed epoch plan");
  const int64_t ps = ds->page_size;
  if (b == 0) {   // epoch start: the reference's install() starts from an empty cache (reader.py:196-208)
    if (PP.phys < P.phys_needed) {
      for (int k = 0; k < kStreams; ++k) CK(cudaStreamSynchronize(L->comp_st[k]));
      CK(cudaStreamSynchronize(L->copy_st));
      if (PP.d_pool) CK(cudaFree(PP.d_pool));
      PP.d_pool = nullptr;
      CK(cudaMalloc(&PP.d_pool, (size_t)P.phys_needed * ps));
      PP.phys = P.phys_needed;
      PP.page_in.assign((size_t)PP.phys, -1);
      PP.user_ring.assign((size_t)PP.phys, -1);
      PP.user_serial.assign((size_t)PP.phys, 0);
    }
    for (int64_t ph = 0; ph < PP.phys; ++ph)
      if (PP.page_in[ph] >= 0) { PP.slot_of[PP.page_in[ph]] = -1; PP.page_in[ph] = -1; }
    PP.free_list.clear();
    for (int64_t ph = PP.phys - 1; ph >= 0; --ph) PP.free_list.push_back(ph);
  }
  int64_t reloads = 0;
  for (int64_t k = k0; k < k1; ++k) {
    const int pos = (int)(k - k0);
    for (int64_t t = P.trace_off[k]; t < P.trace_off[k + 1]; ++t) {
      const PageStep& st = P.trace[t];
      if (st.fetch) {
        int64_t ph;
        if (st.victim >= 0) {
          const int64_t vp = PP.slot_of[st.victim];
          PP.slot_of[st.victim] = -1;
          PP.page_in[vp] = -1;
          if (st.deferred) {
            deferred.push_back(vp);
            if (PP.free_list.empty()) return fail(BBX_INVALID_ARGUMENT, "page pool: no spare page slot");
            ph = PP.free_list.back();
            PP.free_list.pop_back();
          } else {
            ph = vp;
          }
        } else {
          if (PP.free_list.empty()) return fail(BBX_INVALID_ARGUMENT, "page pool: no free page slot");
          ph = PP.free_list.back();
          PP.free_list.pop_back();
        }
        if (int r = fetch_page(L, st.page, ph)) return r;
        PP.slot_of[st.page] = ph;
        PP.page_in[ph] = st.page;
        reloads += st.reload;
      }
      read_slots.push_back(PP.slot_of[st.page]);
    }
    const int64_t i = S.idx[pos];
    if (i < 0 || i >= ds->num_samples) continue;
    for (size_t p = 0; p < L->plans.size(); ++p) {
      const Plan& pl = L->plans[p];
      if (pl.scalar) continue;
      const Field& f = ds->fields[pl.field_index];
      uint64_t off, len;
      if (f.info.kind == 4) { const ImageCell c = image_cell(ds, i, f); off = c.offset; len = c.length; }
      else { off = u64_cell(ds, i, f); len = (uint64_t)f.array_nbytes; }
      if (!len || (int64_t)off < ds->heap_offset || off + len > (uint64_t)ds->alloc_table_offset) continue;
      const int64_t q = ((int64_t)off - ds->heap_offset) / ps;
      if (q != ((int64_t)(off + len - 1) - ds->heap_offset) / ps || PP.slot_of[q] < 0) continue;
      addr[p][pos] = PP.d_pool + (size_t)PP.slot_of[q] * ps + ((int64_t)off - ds->heap_offset - q * ps);
    }
  }
  {
    std::lock_guard<std::mutex> g(L->stats_mu);
    L->stats.page_reloads += reloads;
  }
  return BBX_OK;
}

// A profiled batch's kernel window (events k0 / k1 on its compute stream), added
// to the stats once its events have completed.  The host never waits for them on
// the batch's own step (that would drain the GPU queue, and the next profiled
// launch would then be timed from an idle GPU, host launch latency included): they
// are read when the slot is reused, or by bbx_loader_get_stats.  Caller holds
// stats_mu; k1 has completed.
static void collect_timing(bbx_loader* L, Slot& S) {
  if (!S.timed) return;
  S.timed = false;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, S.k0, S.k1) != cudaSuccess) { cudaGetLastError(); return; }
  float a0 = 0.f, a1 = 0.f;   // absolute k0 / k1 against the loader's reference event
  if (L->t_ref && cudaEventElapsedTime(&a0, L->t_ref, S.k0) == cudaSuccess &&
      cudaEventElapsedTime(&a1, L->t_ref, S.k1) == cudaSuccess) {
    if (L->prof_every == 1 && L->last_k1_ms >= 0.f && a0 > L->last_k1_ms) {
      L->stats.gap_seconds += (a0 - L->last_k1_ms) * 1e-3;
      float ah = 0.f;   // of that gap: the part spent waiting for this batch's H2D (host-late staging)
      if (S.h2d_timed && cudaEventElapsedTime(&ah, L->t_ref, S.h2d_t) == cudaSuccess && ah > L->last_k1_ms)
        L->stats.h2d_late_seconds += (std::min(ah, a0) - L->last_k1_ms) * 1e-3;
    }
    L->last_k1_ms = a1;
  }
  L->stats.kernel_seconds += ms * 1e-3;
  L->stats.timed_batches += 1;
  L->stats.kernel_timed += S.timed_launches;
  L->stats.kernel_bytes += S.timed_bytes;
}

static int process_slot(bbx_loader* L, int s) {
  Slot& S = L->slots[s];
  const bbx_dataset* ds = L->ds;
  const int count = S.count;
  const bool resident = L->payload_dev != nullptr;   // HBM heap or zero-copy: no payload staging
  CK(cudaSetDevice(L->device));
  int64_t zc_bytes = 0;
  // the pinned slot may still be the source of the previous H2D
  if (S.used) CK(cudaEventSynchronize(S.h2d_on_compute ? S.done : S.h2d_done));
  if (S.used) {   // the slot's previous batch: its profiling window, if it had one
    CK(cudaEventSynchronize(S.done));
    std::lock_guard<std::mutex> g(L->stats_mu);
    collect_timing(L, S);
  }
  ++S.serial;
  S.n_gcopies = 0;
  S.herr = HostErr{};
  S.plan_has_rle.assign(L->plans.size(), 0);
  S.plan_has_jpeg.assign(L->plans.size(), 0);
  S.jpeg_total_int.assign(L->plans.size(), 0);
  S.jpeg_total_blk.assign(L->plans.size(), 0);
  S.jpeg_max_quads.assign(L->plans.size(), 0);
  S.jpeg_max_blocks.assign(L->plans.size(), 0);
  uint8_t* H = S.h_stage;
  std::memcpy(H + L->idx_off, S.idx.data(), (size_t)count * 8);
  for (int64_t pos = 0; pos < count; ++pos) {
    int64_t i = S.idx[pos];
    if (i < 0 || i >= ds->num_samples) {
      if (S.herr.pos < 0) {
        S.herr.pos = pos; S.herr.code = BBX_INDEX_OUT_OF_RANGE;
        char buf[128];
        std::snprintf(buf, sizeof buf, "sample %lld out of range [0, %lld)", (long long)i, (long long)ds->num_samples);
        S.herr.msg = buf;
      }
      reinterpret_cast<int64_t*>(H + L->idx_off)[pos] = 0;   // keep device gathers in bounds
    }
  }
  // page pool: this batch's fetches, and where each payload sits in the pool
  std::vector<std::vector<const uint8_t*>> pool_addr;
  std::vector<int64_t> pool_read, pool_deferred;
  if (L->pp.capacity) {
    pool_addr.assign(L->plans.size(), std::vector<const uint8_t*>((size_t)count, nullptr));
    if (int r = page_batch(L, S, count, pool_addr, pool_read, pool_deferred)) return r;
  }
  const uint8_t* stage_dev = S.d_stage + L->pay_base;   // device address of the staged payload region
  // descriptors + payload plan (serial: ~100 ns per sample per field)
  struct Copy { const uint8_t* src; uint8_t* dst; uint32_t row_bytes, rows, src_stride, dst_stride; };
  std::vector<Copy> copies;
  struct JParse { int plan; int pos; int64_t idx; uint64_t off; uint32_t len; };
  std::vector<JParse> jparse;
  // interval starts of this batch's JPEG samples, per plan and position: the
  // loader cache's entry, or (no cache / duplicate index) a slot-local vector
  std::vector<std::vector<const std::vector<uint32_t>*>> jst(L->plans.size());
  std::vector<std::vector<uint32_t>> jlocal;
  if (!resident) copies.reserve((size_t)count * L->plans.size());
  double t0 = (double)std::chrono::steady_clock::now().time_since_epoch().count() * 1e-9;
  // one compact payload region for every plan: [pay_base, cursor)
  const size_t pay_base = L->pay_base;
  size_t cursor = pay_base;
  // descriptors (RNG draws + cell checks) of large batches whose chains draw
  // RandomResizedCrop windows (~60 ns per sample: log / exp / sqrt per attempt) are
  // filled on the staging pool: the pipeline thread is otherwise the bound of an
  // HBM-resident configs[1] batch (measured 31.5 -> 25 us per 512).  Cheaper chains
  // (~20 ns per sample) stay serial: waking the pool costs more (configs[0]: 10 vs 22 us).
  constexpr int kDescChunk = 64;
  bool rrc_draws = false;
  for (const Plan& pl : L->plans)
    for (const Draw& dr : pl.draws) rrc_draws = rrc_draws || dr.kind == BBX_OP_RRC;
  const bool par_desc = rrc_draws && count >= L->par_desc_min && count > kDescChunk;
  std::vector<uint64_t> d_off;
  std::vector<uint32_t> d_len;
  std::vector<uint8_t> d_ok;
  for (size_t p = 0; p < L->plans.size(); ++p) {
    const Plan& pl = L->plans[p];
    if (pl.scalar) continue;
    uint8_t* dblk = H + L->desc_off[p];
    const bool image = ds->fields[pl.field_index].info.kind == 4;
    JpegDesc* jds = pl.field_has_jpeg ? reinterpret_cast<JpegDesc*>(H + L->jpeg_off[p]) : nullptr;
    if (jds) { std::memset(jds, 0, sizeof(JpegDesc) * count); jst[p].assign(count, nullptr); }
    // HBM-resident payloads need nothing from the per-position pass below but the
    // payload offset and the RLE flag: the pool sets them too, and that pass is skipped
    const bool finish_in_pool = par_desc && resident && !L->zc && pool_addr.empty() && !pl.field_has_jpeg;
    if (par_desc) {
      d_off.assign(count, 0); d_len.assign(count, 0); d_ok.assign(count, 0);
      const int64_t nchunk = (count + kDescChunk - 1) / kDescChunk;
      std::vector<HostErr> cerr((size_t)nchunk);
      std::vector<uint8_t> crle((size_t)nchunk, 0);
      L->pool->parallel_for(nchunk, [&](int64_t c) {
        for (int pos = (int)(c * kDescChunk), e = std::min(count, pos + kDescChunk); pos < e; ++pos) {
          const int64_t i = S.idx[pos];
          uint8_t* desc = dblk + (size_t)pos * pl.dev.desc_stride;
          if (i < 0 || i >= ds->num_samples) {
            if (finish_in_pool) {
              std::memset(desc, 0, pl.dev.desc_stride);
              reinterpret_cast<SampleDesc*>(desc)->skip = 1;
            }
            continue;
          }
          d_ok[pos] = fill_desc(ds, pl, i, S.seed, S.epoch, desc, &d_off[pos], &d_len[pos], cerr[c], pos, (int)p) ? 1 : 0;
          if (finish_in_pool && d_ok[pos]) {
            SampleDesc* d = reinterpret_cast<SampleDesc*>(desc);
            d->src = d_off[pos];                        // absolute file offset; base = heap - heap_offset
            if (d->codec == CODEC_RLE && image) crle[c] = 1;
          }
        }
      });
      for (const HostErr& e : cerr)   // chunks are in position order: the first error is the lowest
        if (e.pos >= 0) {
          if (S.herr.pos < 0 || e.pos < S.herr.pos || (e.pos == S.herr.pos && e.plan < S.herr.plan)) S.herr = e;
          break;
        }
      if (finish_in_pool) {
        for (uint8_t f : crle) S.plan_has_rle[p] |= f;
        continue;
      }
    }
    for (int pos = 0; pos < count; ++pos) {
      int64_t i = S.idx[pos];
      uint8_t* desc = dblk + (size_t)pos * pl.dev.desc_stride;
      if (i < 0 || i >= ds->num_samples) {
        std::memset(desc, 0, pl.dev.desc_stride);
        reinterpret_cast<SampleDesc*>(desc)->skip = 1;
        continue;
      }
      uint64_t off = 0;
      uint32_t len = 0;
      bool ok;
      if (par_desc) { ok = d_ok[pos] != 0; off = d_off[pos]; len = d_len[pos]; }
      else ok = fill_desc(ds, pl, i, S.seed, S.epoch, desc, &off, &len, S.herr, pos, (int)p);
      SampleDesc* d = reinterpret_cast<SampleDesc*>(desc);
      if (!ok) continue;
      if (d->codec == CODEC_RLE && ds->fields[pl.field_index].info.kind == 4) S.plan_has_rle[p] = 1;
      if (image && d->codec == CODEC_JPEG) {   // header: from the cache, else parsed on the pool below
        if (L->jpeg_cache && pl.jcached[i]) { jds[pos] = pl.jcache[i]; jst[p][pos] = &pl.jstarts[i]; }
        else jparse.push_back({(int)p, pos, i, off, len});
        S.plan_has_jpeg[p] = 1;
      }
      if (!pool_addr.empty() && pool_addr[p][pos]) {   // in the HBM page pool (offset from the staged base)
        d->src = (uint64_t)(pool_addr[p][pos] - stage_dev);
        continue;
      }
      if (resident) {
        d->src = off;                                   // absolute file offset; base = heap - heap_offset
        if (L->zc) {                                    // bytes the kernels will pull over PCIe
          if (image && d->codec == CODEC_RAW) {
            int y0, y1, x0, x1;
            read_window(pl.dev, d, reinterpret_cast<const int32_t*>(desc + kDescHeader), &y0, &y1, &x0, &x1);
            zc_bytes += (int64_t)(y1 - y0) * (x1 - x0) * d->c;
          } else {
            zc_bytes += len;
          }
        }
        continue;
      }
      d->src = cursor - pay_base;                       // relative to the payload region
      if (image && d->codec == CODEC_RAW && L->window_staging) {
        int y0, y1, x0, x1;
        read_window(pl.dev, d, reinterpret_cast<const int32_t*>(desc + kDescHeader), &y0, &y1, &x0, &x1);
        const uint32_t wb = (uint32_t)(x1 - x0) * d->c, wr = (uint32_t)(y1 - y0);
        // staged rows start 16-byte aligned (the gather streams whole 16-B chunks);
        // worth it below 90 % of the payload, and never above the sample's staging share
        const uint32_t ws = (wb + 15) & ~15u;
        if ((uint64_t)wb * wr * 10 < (uint64_t)len * 9 && (uint64_t)ws * wr <= ((uint64_t)len + 15) / 16 * 16) {
          d->flags |= kDescWindowed;
          d->wstride = ws; d->wy0 = (uint16_t)y0; d->wx0 = (uint16_t)x0;
          if (wb && wr)
            copies.push_back({ds->map + off + ((uint64_t)y0 * d->w + x0) * d->c, H + cursor, wb, wr,
                              (uint32_t)d->w * d->c, ws});
          cursor += (size_t)ws * wr;
          continue;
        }
      }
      if (len) copies.push_back({ds->map + off, H + cursor, len, 1, len, len});
      cursor += ((size_t)len + 15) / 16 * 16;
    }
  }
  // JPEG headers not seen before: parse on the pool (tables registered under a mutex)
  if (!jparse.empty()) {
    std::vector<HostErr> jerr(jparse.size());
    jlocal.assign(jparse.size(), {});
    // the cache entry of a sample is written by its first occurrence in the batch
    // only (a padded distributed tail can repeat an index)
    std::vector<char> first(jparse.size(), 1);
    if (L->jpeg_cache) {
      std::unordered_map<int64_t, size_t> seen;
      for (size_t q = 0; q < jparse.size(); ++q)
        if (!seen.emplace(jparse[q].idx * 64 + jparse[q].plan, q).second) first[q] = 0;
    }
    L->pool->parallel_for((int64_t)jparse.size(), [&](int64_t q) {
      const JParse& j = jparse[q];
      Plan& pl = L->plans[j.plan];
      uint8_t* desc = H + L->desc_off[j.plan] + (size_t)j.pos * pl.dev.desc_stride;
      JpegDesc* jd = reinterpret_cast<JpegDesc*>(H + L->jpeg_off[j.plan]) + j.pos;
      if (jpeg_prepare(L, pl, ds->map + j.off, j.len, reinterpret_cast<SampleDesc*>(desc), jd, &jlocal[q], jerr[q],
                       j.pos, j.plan)) {
        if (L->jpeg_cache && first[q]) { pl.jcache[j.idx] = *jd; pl.jstarts[j.idx] = jlocal[q]; pl.jcached[j.idx] = 1; }
      }
    });
    for (size_t q = 0; q < jparse.size(); ++q) jst[jparse[q].plan][jparse[q].pos] = &jlocal[q];
    for (const HostErr& e : jerr)
      if (e.pos >= 0 && (S.herr.pos < 0 || e.pos < S.herr.pos || (e.pos == S.herr.pos && e.plan < S.herr.plan)))
        S.herr = e;
  }
  // JPEG: interval / block prefixes of each plan's batch (J2/J3 thread maps)
  for (size_t p = 0; p < L->plans.size(); ++p) {
    if (!S.plan_has_jpeg[p]) continue;
    const Plan& pl = L->plans[p];
    uint8_t* jb = H + L->jpeg_off[p];
    JpegDesc* jds = reinterpret_cast<JpegDesc*>(jb);
    uint32_t* ipre = reinterpret_cast<uint32_t*>(jb + jpeg_iprefix_off(L->batch));
    uint64_t* bpre = reinterpret_cast<uint64_t*>(jb + jpeg_bprefix_off(L->batch));
    uint32_t* starts = reinterpret_cast<uint32_t*>(jb + jpeg_block_bytes(L->batch));
    const uint8_t* dblk = H + L->desc_off[p];
    uint32_t ti = 0;
    uint64_t tb = 0;
    int32_t mq = 0;
    uint32_t mb = 0;
    for (int pos = 0; pos < count; ++pos) {
      JpegDesc& J = jds[pos];
      const SampleDesc* d = reinterpret_cast<const SampleDesc*>(dblk + (size_t)pos * pl.dev.desc_stride);
      if (d->skip) J.n_int = 0;
      if (J.n_int == 0) J.n_blocks = 0;
      if (J.n_int) {   // region of interest: the pixels this sample's chain reads
        int y0, y1, x0, x1;
        read_window(pl.dev, d, reinterpret_cast<const int32_t*>(dblk + (size_t)pos * pl.dev.desc_stride + kDescHeader),
                    &y0, &y1, &x0, &x1);
        if (!L->jpeg_roi) { y0 = 0; y1 = d->h; x0 = 0; x1 = d->w; }
        J.win[0] = (uint16_t)y0; J.win[1] = (uint16_t)y1; J.win[2] = (uint16_t)x0; J.win[3] = (uint16_t)x1;
      }
      J.int_base = ti; J.blk_base = tb;
      ipre[pos] = ti; bpre[pos] = tb;
      if (J.n_int) std::memcpy(starts + ti, jst[p][pos]->data(), (size_t)J.n_int * 4);
      ti += J.n_int; tb += J.n_blocks;
      if (J.n_int) {
        mq = std::max(mq, (int32_t)d->h);
        mb = std::max(mb, J.n_blocks);
      }
    }
    ipre[count] = ti; bpre[count] = tb;
    S.jpeg_total_int[p] = ti; S.jpeg_total_blk[p] = tb; S.jpeg_max_quads[p] = mq; S.jpeg_max_blocks[p] = mb;
    if (ti == 0) S.plan_has_jpeg[p] = 0;
  }
  {   // new JPEG tables: append-only upload ahead of this slot's H2D (same copy stream)
    JpegTables& T = L->jt;
    if (T.n_huff > T.up_huff) {
      CK(cudaMemcpyAsync(T.d_huff + T.up_huff, T.h_huff + T.up_huff, sizeof(JHuff) * (T.n_huff - T.up_huff),
                         cudaMemcpyHostToDevice, L->copy_st));
      T.up_huff = T.n_huff;
    }
    if (T.n_quant > T.up_quant) {
      CK(cudaMemcpyAsync(T.d_quant + T.up_quant, T.h_quant + T.up_quant, sizeof(JQuant) * (T.n_quant - T.up_quant),
                         cudaMemcpyHostToDevice, L->copy_st));
      T.up_quant = T.n_quant;
    }
  }
  // gather mode: mmap page cache -> pinned slot (row segments for windows)
  if (!copies.empty() && L->direct_io) {   // Direct: pread each payload (whole, unwindowed)
    std::atomic<int> io_err{0};
    L->pool->parallel_for((int64_t)copies.size(), [&](int64_t k) {
      const Copy& c = copies[k];
      if (L->read_latency_ns > 0) {
        const auto until = std::chrono::steady_clock::now() + std::chrono::nanoseconds(L->read_latency_ns);
        while (std::chrono::steady_clock::now() < until) {}
      }
      const off_t at = (off_t)(c.src - ds->map);
      size_t done = 0;
      while (done < c.row_bytes) {
        const ssize_t r = ::pread(ds->fd, c.dst + done, c.row_bytes - done, at + (off_t)done);
        if (r <= 0) { io_err = 1; break; }
        done += (size_t)r;
      }
    });
    if (io_err) return fail(BBX_INVALID_FILE, "%s: short read", ds->path.c_str());
    std::lock_guard<std::mutex> g(L->stats_mu);
    L->stats.io_reads += (int64_t)copies.size();
  } else if (!copies.empty() && L->zcg) {   // the device gathers them: only the copy list goes up
    GatherCopy* g = reinterpret_cast<GatherCopy*>(H + L->gcopy_off);
    const uint8_t* hb = ds->map + ds->heap_offset;
    for (size_t k = 0; k < copies.size(); ++k) {
      const Copy& c = copies[k];
      g[k] = GatherCopy{(uint64_t)(c.src - hb), (uint64_t)(c.dst - H), c.row_bytes, c.rows, c.src_stride, c.dst_stride};
    }
    S.n_gcopies = (int)copies.size();
  } else if (!copies.empty()) {
    const uint8_t* map_end = ds->map + ds->map_len;
    // small payloads (CIFAR-sized: ~3 KB) are claimed several at a time, ~16 KB per claim
    // (A/B, configs[0] e2e: per-item claims 4.3-5.1, 16 KB 5.2-5.7, 64 KB 4.4-5.5 M img/s;
    // the larger payloads of configs[1] / [2] keep one copy per claim)
    constexpr int64_t kGatherGrainBytes = 16384;
    const int64_t per_copy = (int64_t)(cursor - pay_base) / (int64_t)copies.size();
    const int64_t grain = std::min<int64_t>(64, std::max<int64_t>(1, kGatherGrainBytes / std::max<int64_t>(per_copy, 1)));
    L->pool->parallel_for((int64_t)copies.size(), [&](int64_t k) {
      const Copy& c = copies[k];
      gather_rows(c.dst, c.dst_stride, c.src, c.src_stride, c.row_bytes, c.rows, map_end);
    }, grain);
  }
  double t1 = (double)std::chrono::steady_clock::now().time_since_epoch().count() * 1e-9;
  // consecutive batches go to alternating compute streams: one batch's kernels can
  // fill the SMs that the previous batch's tail (e.g. the last Huffman lanes) leaves idle.
  // The stream is a function of the slot (consecutive batches use consecutive slots), so
  // each slot's captured graph is reused by every later iterator of the loader.
  const int sk = s % L->nstreams;
  ++L->batch_seq;
  cudaStream_t cs = L->comp_st[sk];
  const size_t bytes = resident ? L->desc_bytes : cursor;
  // A resident RAW / RLE / array batch uploads only its indices + descriptors (tens of KB): that copy
  // goes on the compute stream itself, ordered after the slot's previous kernels by
  // the stream (or one event wait when they ran on the other stream) -- three fewer
  // API calls on the pipeline thread, which bounds the small-image legs.  Payload
  // batches copy on the copy stream so the H2D overlaps the previous batches' kernels.
  bool jpeg_plan = false;   // JPEG tables are uploaded on the copy stream ahead of its H2D
  for (const Plan& pl : L->plans) jpeg_plan = jpeg_plan || pl.field_has_jpeg;
  const bool h2d_compute = resident && !jpeg_plan && !(L->profiling && L->prof_every == 1);
  // profiling: every prof_every-th batch gets the CUDA-event window (sampling keeps
  // the events' own cost off most batches)
  const bool prof = L->profiling && (L->prof_seq++ % (uint64_t)L->prof_every) == 0;
  bool any_status = false;   // device-detected sample errors to read back (RLE / JPEG)
  for (size_t p = 0; p < L->plans.size(); ++p) any_status = any_status || S.plan_has_rle[p] || S.plan_has_jpeg[p];
  int launches = 0;
  int64_t kbytes = 0, klaunch = 0, d2h = 0;
  bool wait_release;   // the consumer released the slot since its last batch: order after that
  {
    std::lock_guard<std::mutex> g(L->mu);
    wait_release = S.released_pending;
    S.released_pending = false;
  }
  // The batch's stream work: H2D, waits, kernels, status read-back, `done` record.
  // cap: recorded into a CUDA graph instead of issued (stream capture).
  auto enqueue = [&](bool cap) -> int {
    if (h2d_compute) {
      if (!cap && S.used && S.last_stream != sk) CK(cudaStreamWaitEvent(cs, S.done, 0));
      CK(cudaMemcpyAsync(S.d_stage, S.h_stage, bytes, cudaMemcpyHostToDevice, cs));
      S.h2d_timed = false;
    } else {
      // H2D on the copy stream (after the previous kernels reading d_stage); a
      // zero-copy-gather batch uploads only its descriptors and copy list
      if (S.used) CK(cudaStreamWaitEvent(L->copy_st, S.done, 0));
      CK(cudaMemcpyAsync(S.d_stage, S.h_stage, S.n_gcopies ? L->pay_base : bytes, cudaMemcpyHostToDevice, L->copy_st));
      CK(cudaEventRecord(S.h2d_done, L->copy_st));
      S.h2d_timed = false;
      if (L->profiling && L->prof_every == 1) {   // idle-gap attribution needs every batch timed
        if (!S.h2d_t) CK(cudaEventCreate(&S.h2d_t));
        CK(cudaEventRecord(S.h2d_t, L->copy_st));
        S.h2d_timed = true;
      }
      CK(cudaStreamWaitEvent(cs, S.h2d_done, 0));
    }
    S.h2d_on_compute = h2d_compute;
    S.last_stream = sk;
    // a captured batch always waits on the slot's release event (a no-op when the
    // consumer has not recorded a newer one): the graph is replayed every batch
    if (cap) CK(cudaStreamWaitEvent(cs, S.release, cudaEventWaitExternal));
    else if (wait_release) CK(cudaStreamWaitEvent(cs, S.release, 0));
    launches = 0;
    kbytes = 0; klaunch = 0;
    if (prof && !L->t_ref) {
      CK(cudaEventCreate(&L->t_ref));
      CK(cudaEventRecord(L->t_ref, cs));
    }
    if (prof) CK(cudaEventRecord(S.k0, cs));
    if (S.n_gcopies) {
      if (launch_host_gather(ds->h_heap_dev, (uint64_t)(ds->alloc_table_offset - ds->heap_offset), S.d_stage,
                             reinterpret_cast<const GatherCopy*>(S.d_stage + L->gcopy_off), S.n_gcopies, cs))
        return fail(BBX_CUDA_ERROR, "gather launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      ++launches;
    }
    d2h = 0;
    ScalarArgs SA{};
    SA.idx = reinterpret_cast<const int64_t*>(S.d_stage + L->idx_off);
    SA.count = count;
    // up to 16 scalar fields ride along with the first image plan's K1 launch (the
    // column walker's copy warp, or tile 0 of the tile kernel, gathers them);
    // otherwise, or beyond that, scalar_gather_kernel
    int n_scalar = 0, fused_plan = -1;
    for (const Plan& pl : L->plans) n_scalar += pl.scalar ? 1 : 0;
    if (n_scalar > 0 && n_scalar <= 16 && count > 0)   // an image plan's K1 (either variant) carries them
      for (size_t p = 0; p < L->plans.size(); ++p)
        if (!L->plans[p].scalar && L->plans[p].dev.src_kind != SRC_ARRAY) { fused_plan = (int)p; break; }
    if (fused_plan >= 0)
      for (const Plan& pl : L->plans)
        if (pl.scalar) {
          SA.cols[SA.n_fields] = pl.d_col;
          SA.outs[SA.n_fields] = reinterpret_cast<uint64_t*>(pl.outs[s]);
          ++SA.n_fields;
        }
    for (size_t p = 0; p < L->plans.size(); ++p) {
      Plan& pl = L->plans[p];
      if (pl.scalar) {
        if (fused_plan >= 0) continue;
        SA.cols[SA.n_fields] = pl.d_col;
        SA.outs[SA.n_fields] = reinterpret_cast<uint64_t*>(pl.outs[s]);
        ++SA.n_fields;
        if (SA.n_fields == 16) { if (launch_scalar_gather(SA, cs)) return fail(BBX_CUDA_ERROR, "scalar gather launch failed"); ++launches; SA.n_fields = 0; }
        continue;
      }
      LaunchArgs A{};
      A.desc = S.d_stage + L->desc_off[p];
      A.payload = resident ? (const uint8_t*)(L->payload_dev - ds->heap_offset) : (const uint8_t*)(S.d_stage + L->pay_base);
      A.scratch = pl.d_scratch.empty() ? nullptr : pl.d_scratch[s];
      A.tables = pl.d_tables.empty() ? nullptr : pl.d_tables[s];
      A.lut = pl.d_lut;
      A.out = pl.outs[s];
      A.status = S.d_status + (size_t)p * L->batch;
      A.count = count;
      if ((int)p == fused_plan) A.sc = SA;
      A.ticket = pl.d_ticket[sk];
      if (count == 0) continue;
      if (S.plan_has_rle[p]) {
        if (launch_rle_expand(pl.dev, A, cs)) return fail(BBX_CUDA_ERROR, "rle launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        ++launches;
      }
      if (S.plan_has_jpeg[p]) {
        JpegArgs J{};
        const uint8_t* jb = S.d_stage + L->jpeg_off[p];
        J.desc = A.desc; J.desc_stride = pl.dev.desc_stride; J.payload = A.payload;
        J.jd = reinterpret_cast<const JpegDesc*>(jb);
        J.int_prefix = reinterpret_cast<const uint32_t*>(jb + jpeg_iprefix_off(L->batch));
        J.blk_prefix = reinterpret_cast<const uint64_t*>(jb + jpeg_bprefix_off(L->batch));
        J.starts = reinterpret_cast<const uint32_t*>(jb + jpeg_block_bytes(L->batch));
        J.coef = pl.d_coef[sk]; J.planes = pl.d_planes[sk];
        J.scratch = A.scratch; J.scratch_bytes = pl.dev.scratch_bytes;
        J.huff = L->jt.d_huff; J.quant = L->jt.d_quant; J.n_huff = L->jt.n_huff; J.status = A.status; J.count = count;
        J.coef_zeroed = 1;
        J.total_int = S.jpeg_total_int[p]; J.total_blocks = S.jpeg_total_blk[p]; J.max_quads = S.jpeg_max_quads[p];
        J.max_blocks = S.jpeg_max_blocks[p];
        if (launch_jpeg(J, cs)) return fail(BBX_CUDA_ERROR, "jpeg launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        launches += 4;
      }
      int rc = pl.dev.src_kind == SRC_ARRAY ? launch_array(pl.dev, A, cs) : launch_image(pl.dev, A, cs);
      if (prof) {   // algorithmic bytes: source bytes the chain needs + output bytes
        ++klaunch;
        const uint8_t* dblk = H + L->desc_off[p];
        for (int pos = 0; pos < count; ++pos) {
          const SampleDesc* d = reinterpret_cast<const SampleDesc*>(dblk + (size_t)pos * pl.dev.desc_stride);
          if (d->skip) continue;
          const int32_t* prm = reinterpret_cast<const int32_t*>(dblk + (size_t)pos * pl.dev.desc_stride + kDescHeader);
          int64_t rd;
          if (pl.dev.src_kind == SRC_RESAMPLE) rd = (int64_t)prm[2] * prm[3] * pl.dev.channels;
          else if (pl.dev.src_kind == SRC_ARRAY) rd = std::min<int64_t>(d->len, pl.dev.out_sample_elems * pl.dev.src_elem);
          else rd = std::min<int64_t>(d->len, pl.dev.out_sample_elems);
          kbytes += rd + pl.out_sample_bytes;
        }
      }
      if (rc) return fail(BBX_CUDA_ERROR, "kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      launches += (pl.dev.src_kind == SRC_ARRAY || pl.dev.cw) ? 1 : 2;   // K1 = prologue + tiles (column walker: one kernel)
    }
    if (prof) CK(cudaEventRecord(S.k1, cs));
    {
      std::lock_guard<std::mutex> g(L->stats_mu);   // read by bbx_loader_get_stats on the consumer thread
      S.timed = prof;
      S.timed_launches = klaunch;
      S.timed_bytes = kbytes;
    }
    if (SA.n_fields && count && fused_plan < 0) {
      if (launch_scalar_gather(SA, cs)) return fail(BBX_CUDA_ERROR, "scalar gather launch failed");
      ++launches;
    }
    if (any_status) {
      size_t nb = sizeof(SampleStatus) * L->batch * L->plans.size();
      CK(cudaMemcpyAsync(S.h_status, S.d_status, nb, cudaMemcpyDeviceToHost, cs));
      d2h += (int64_t)nb;
    }
    if (cap) CK(cudaEventRecordWithFlags(S.done, cs, cudaEventRecordExternal));
    else CK(cudaEventRecord(S.done, cs));
    return 0;
  };
  // A full-size resident batch without per-sample device status has the same stream
  // work every time: it is captured once per (slot, compute stream) into a CUDA graph
  // and replayed with one cudaGraphLaunch (the host pipeline thread -- ~5 API calls
  // and 1-2 launches per batch otherwise -- bounds the small-image legs).
  const bool graph_ok = L->use_graphs && h2d_compute && !prof && !any_status && count == L->batch && !L->pp.capacity;
  if (graph_ok && S.gexec[sk]) {
    if (S.used && S.last_stream != sk) CK(cudaStreamWaitEvent(cs, S.done, 0));
    CK(cudaGraphLaunch(S.gexec[sk], cs));
    S.h2d_on_compute = true;
    S.last_stream = sk;
    launches = S.glaunches[sk];
    S.timed = false;
  } else if (graph_ok) {
    if (S.used && S.last_stream != sk) CK(cudaStreamWaitEvent(cs, S.done, 0));
    bool captured = false;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      const int r = enqueue(true);
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(cs, &g);
      if (r == 0 && ec == cudaSuccess && g && cudaGraphInstantiate(&S.gexec[sk], g, 0) == cudaSuccess) {
        captured = true;
        S.glaunches[sk] = launches;
      }
      if (g) cudaGraphDestroy(g);
    }
    if (captured) {
      CK(cudaGraphLaunch(S.gexec[sk], cs));
    } else {                                           // capture unsupported here: plain launches from now on
      cudaGetLastError();
      S.gexec[sk] = nullptr;
      L->use_graphs = false;
      if (int r = enqueue(false)) return r;
    }
  } else {
    if (int r = enqueue(false)) return r;
  }
  S.used = true;
  if (L->pp.capacity) {   // the pool slots this batch reads are recycled only after S.done
    PagePool& PP = L->pp;
    for (int64_t ph : pool_read) { PP.user_ring[ph] = s; PP.user_serial[ph] = S.serial; }
    for (int64_t ph : pool_deferred) { PP.user_ring[ph] = s; PP.user_serial[ph] = S.serial; PP.free_list.push_back(ph); }
    std::lock_guard<std::mutex> g(L->mu);
    PagePlan& P = PP.plans.front();
    if (++P.next == (int32_t)P.batch_off.size() - 1) PP.plans.pop_front();
  }
  {
    std::lock_guard<std::mutex> g(L->stats_mu);
    L->stats.batches += 1;
    L->stats.samples += count;
    // zero-copy gather: the descriptors go by DMA, the payload rows by the gather kernel's PCIe reads
    L->stats.h2d_bytes += (int64_t)(S.n_gcopies ? L->pay_base : bytes);
    if (S.n_gcopies) zc_bytes += (int64_t)(bytes - L->pay_base);
    L->stats.d2h_bytes += d2h;
    L->stats.kernel_launches += launches;
    L->stats.stage_seconds += t1 - t0;
    L->stats.zero_copy_bytes += zc_bytes;
  }
  return BBX_OK;
}

// codecs.decode_image for one JPEG blob: the batch decoder (J2-J4) run on a
// batch of one, writing the (h, w, c) result straight into out_dev.
static int jpeg_decode_one(int h, int w, int c, const uint8_t* pay, int64_t len, uint8_t* out_dev, int device) {
  if (len < 4 || len > 0xFFFFFFFFll) return fail(BBX_CORRUPT_PAYLOAD, "jpeg: missing SOI marker");
  if (h > 65535 || w > 65535 || c > 255) return fail(BBX_SCHEMA_MISMATCH, "image dims too large");
  CK(cudaSetDevice(device));
  bbx_loader L;                                  // only its table registry is used
  std::vector<JHuff> hh(kJpegMaxHuff);
  std::vector<JQuant> hq(kJpegMaxQuant);
  L.jt.h_huff = hh.data(); L.jt.h_quant = hq.data();
  Plan pl;
  pl.jpeg_blocks_cap = (int64_t)c * (2 * ((h + 15) / 16)) * (2 * ((w + 15) / 16));
  pl.jpeg_int_cap = (int64_t)((h + 7) / 8) * ((w + 7) / 8);
  uint8_t desc[64] = {0};
  SampleDesc* d = reinterpret_cast<SampleDesc*>(desc);
  d->src = 0; d->len = (uint32_t)len; d->h = (uint16_t)h; d->w = (uint16_t)w; d->c = (uint8_t)c; d->codec = CODEC_JPEG;
  JpegDesc J{};
  std::vector<uint32_t> starts;
  HostErr err;
  bool ok = jpeg_prepare(&L, pl, pay, (uint32_t)len, d, &J, &starts, err, 0, 0);
  L.jt.h_huff = nullptr; L.jt.h_quant = nullptr;
  if (!ok) return fail(err.code, "%s", err.msg.c_str());
  J.int_base = 0; J.blk_base = 0;
  J.win[0] = 0; J.win[1] = (uint16_t)h; J.win[2] = 0; J.win[3] = (uint16_t)w;
  // device image: [desc 64][jd][prefixes][payload (+16 pad)][tables][interval starts] then coef, planes, status
  const size_t o_jd = 64, o_ip = o_jd + sizeof(JpegDesc), o_bp = o_ip + 16, o_pay = o_bp + 16;
  const size_t o_hf = (o_pay + len + 16 + 255) / 256 * 256;
  const size_t o_q = o_hf + sizeof(JHuff) * L.jt.n_huff;
  const size_t o_is = (o_q + sizeof(JQuant) * L.jt.n_quant + 255) / 256 * 256;
  const size_t o_cf = (o_is + 4 * (size_t)J.n_int + 16 + 255) / 256 * 256;
  const size_t o_pl = (o_cf + 128 * (size_t)J.n_blocks + 255) / 256 * 256;
  const size_t o_st = (o_pl + 64 * (size_t)J.n_blocks + 255) / 256 * 256;
  const size_t total = o_st + sizeof(SampleStatus);
  std::vector<uint8_t> img(o_cf, 0);
  std::memcpy(img.data(), desc, 64);
  std::memcpy(img.data() + o_jd, &J, sizeof J);
  const uint32_t ip[2] = {0, J.n_int};
  const uint64_t bp[2] = {0, J.n_blocks};
  std::memcpy(img.data() + o_ip, ip, sizeof ip);
  std::memcpy(img.data() + o_bp, bp, sizeof bp);
  std::memcpy(img.data() + o_pay, pay, (size_t)len);
  std::memcpy(img.data() + o_hf, hh.data(), sizeof(JHuff) * L.jt.n_huff);
  std::memcpy(img.data() + o_q, hq.data(), sizeof(JQuant) * L.jt.n_quant);
  std::memcpy(img.data() + o_is, starts.data(), 4 * (size_t)J.n_int);
  uint8_t* dev = nullptr;
  CK(cudaMalloc(&dev, total));
  cudaError_t e = cudaMemcpy(dev, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dev + o_st, 0, sizeof(SampleStatus));
  if (e == cudaSuccess) e = cudaMemset(dev + o_cf, 0, 128 * (size_t)J.n_blocks);
  JpegArgs A{};
  A.desc = dev; A.desc_stride = 64; A.payload = dev + o_pay;
  A.jd = reinterpret_cast<const JpegDesc*>(dev + o_jd);
  A.int_prefix = reinterpret_cast<const uint32_t*>(dev + o_ip);
  A.blk_prefix = reinterpret_cast<const uint64_t*>(dev + o_bp);
  A.starts = reinterpret_cast<const uint32_t*>(dev + o_is);
  A.coef = reinterpret_cast<int16_t*>(dev + o_cf); A.planes = dev + o_pl;
  A.scratch = out_dev; A.scratch_bytes = (int64_t)h * w * c; A.exact_pitch = 1;   // (h, w, c) output, no row padding
  A.huff = reinterpret_cast<const JHuff*>(dev + o_hf); A.quant = reinterpret_cast<const JQuant*>(dev + o_q);
  A.n_huff = L.jt.n_huff;
  A.coef_zeroed = 1;
  A.status = reinterpret_cast<SampleStatus*>(dev + o_st);
  A.count = 1; A.total_int = J.n_int; A.total_blocks = J.n_blocks; A.max_quads = h; A.max_blocks = J.n_blocks;
  int rc = e == cudaSuccess ? launch_jpeg(A, nullptr) : 1;
  SampleStatus st{};
  if (e == cudaSuccess) e = cudaMemcpy(&st, dev + o_st, sizeof st, cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (rc || e != cudaSuccess) return fail(BBX_CUDA_ERROR, "jpeg decode failed: %s", cudaGetErrorString(e));
  if (st.kind == JST_BAD_CODE) return fail(BBX_CORRUPT_PAYLOAD, "jpeg: bad Huffman code in restart interval %lld", (long long)st.value);
  return BBX_OK;
}

static void pipeline_loop(bbx_loader* L) {
  cudaSetDevice(L->device);
  for (;;) {
    int s;
    {
      std::unique_lock<std::mutex> lk(L->mu);
      L->cv.wait(lk, [&] { return L->stop || !L->queue.empty(); });
      if (L->queue.empty()) return;
      s = L->queue.front();
      L->queue.pop_front();
    }
    const auto p0 = std::chrono::steady_clock::now();
    int rc = process_slot(L, s);
    const double pdt = std::chrono::duration<double>(std::chrono::steady_clock::now() - p0).count();
    {
      std::lock_guard<std::mutex> g(L->stats_mu);
      L->stats.pipeline_seconds += pdt;
    }
    {
      std::lock_guard<std::mutex> g(L->mu);
      Slot& S = L->slots[s];
      S.fatal = rc;
      if (rc) S.fatal_msg = last_error();
      S.state = 2;
    }
    L->done_cv.notify_all();
  }
}

}  // namespace bbx

// =================================================================== C ABI
extern "C" {

const char* bbx_last_error(void) { return bbx::last_error(); }
const char* bbx_version(void) { return "bbx-b200 0.1.0 (sm_100a)"; }

bbx_status bbx_dataset_open(const char* path, bbx_dataset** out) {
  if (!path || !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  return (bbx_status)bbx::dataset_open(path, out);
}
void bbx_dataset_close(bbx_dataset* ds) { bbx::dataset_close(ds); }

bbx_status bbx_dataset_header(const bbx_dataset* ds, bbx_header_info* o) {
  if (!ds || !o) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  o->num_samples = ds->num_samples; o->page_size = ds->page_size; o->data_table_offset = ds->data_table_offset;
  o->heap_offset = ds->heap_offset; o->alloc_table_offset = ds->alloc_table_offset;
  o->num_fields = (int32_t)ds->fields.size(); o->row_width = ds->row_width;
  return BBX_OK;
}
bbx_status bbx_dataset_field(const bbx_dataset* ds, int index, bbx_field_info* o) {
  if (!ds || !o || index < 0 || index >= (int)ds->fields.size())
    return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad field index");
  *o = ds->fields[index].info;
  return BBX_OK;
}
bbx_status bbx_dataset_row(const bbx_dataset* ds, int64_t i, uint8_t* out, int32_t out_len) {
  if (!ds || !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (i < 0 || i >= ds->num_samples)
    return (bbx_status)fail(BBX_INDEX_OUT_OF_RANGE, "sample %lld out of range [0, %lld)", (long long)i,
                            (long long)ds->num_samples);
  if (out_len < ds->row_width) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "row buffer too short");
  std::memcpy(out, ds->rows + i * ds->row_width, ds->row_width);
  return BBX_OK;
}
bbx_status bbx_dataset_make_resident(bbx_dataset* ds, int device) {
  if (!ds) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null dataset");
  return (bbx_status)bbx::dataset_make_resident(ds, device);
}
bbx_status bbx_dataset_pin_host(bbx_dataset* ds, int threads) {
  if (!ds) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null dataset");
  if (threads <= 0) threads = (int)std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency()));
  return (bbx_status)bbx::dataset_pin_host(ds, threads);
}
bbx_status bbx_dataset_page_map(const bbx_dataset* ds, int64_t* out) {
  if (!ds || !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  for (int64_t i = 0; i < ds->num_samples; ++i) out[i] = bbx::primary_page(ds, i);
  return BBX_OK;
}

bbx_status bbx_epoch_order(int kind, uint64_t seed, uint64_t epoch, int64_t n, const int64_t* page_map,
                           int64_t batch_size, int64_t* out) {
  if (n > 0 && !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null output");
  return (bbx_status)bbx::epoch_order(kind, seed, epoch, n, page_map, batch_size, out);
}

bbx_status bbx_loader_create(bbx_dataset* ds, int device, int32_t batch_size, int32_t slot_count,
                             int32_t staging_threads, bbx_loader** out) {
  if (!ds || !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (batch_size < 1) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "batch_size must be >= 1");
  if (slot_count < 1) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "slot_count must be >= 1");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return (bbx_status)fail(BBX_CUDA_ERROR, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  auto L = std::make_unique<bbx_loader>();
  L->ds = ds; L->device = device; L->batch = batch_size; L->nslots = slot_count;
  L->slots.resize(slot_count);
  int nt = staging_threads;
  if (nt <= 0) {   // automatic: the host's cores shared by the node's ranks (torchrun LOCAL_WORLD_SIZE)
    unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) hc = std::max(1u, hc / (unsigned)std::max(1, std::atoi(e)));
    // three quarters of them, at most 16: the pipeline thread, the consumer and the CUDA
    // driver's threads keep a core each (A/B on a 16-vCPU box, e2e configs[1] / configs[2]:
    // 8 threads 454k / 1.43M, 12 threads 488k / 1.63M, 16 threads 475k / 1.60M img/s)
    nt = (int)std::min<unsigned>(16, std::max(1u, hc - hc / 4));
  }
  L->local_cpus = gpu_local_cpus(device, &L->numa_node);
  if (!L->local_cpus.empty()) nt = std::min<int>(nt, (int)L->local_cpus.size());
  L->pool = std::make_unique<Pool>(nt);
  L->pool->pin(L->local_cpus);   // staging threads on the GPU's NUMA node
  if ((e = cudaStreamCreateWithFlags(&L->copy_st, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&L->comp_st[0], cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&L->comp_st[1], cudaStreamNonBlocking)) != cudaSuccess)
    return (bbx_status)fail(BBX_CUDA_ERROR, "stream create: %s", cudaGetErrorString(e));
  *out = L.release();
  return BBX_OK;
}

bbx_status bbx_loader_add_field(bbx_loader* L, int32_t field_index, const bbx_op* ops, int32_t n_ops,
                                int32_t* plan_id, int64_t out_shape[4], int32_t* out_ndim, int32_t* out_dtype) {
  if (!L || !ops) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "loader already started");
  cudaSetDevice(L->device);
  Plan pl;
  int rc = plan_compile(L, field_index, ops, n_ops, pl);
  if (rc) return (bbx_status)rc;
  pl.outs.assign(L->nslots, nullptr);
  const Field& f = L->ds->fields[field_index];
  if (pl.dev.src_kind == SRC_ARRAY && !pl.dev.has_remaps_3d) {
    *out_ndim = f.info.ndims;
    for (int k = 0; k < 4; ++k) out_shape[k] = k < f.info.ndims ? f.info.dims[k] : 0;
  } else {
    *out_ndim = 3;
    out_shape[0] = pl.dev.out_h; out_shape[1] = pl.dev.out_w; out_shape[2] = pl.dev.out_c; out_shape[3] = 0;
  }
  *out_dtype = pl.dev.out_dtype;
  *plan_id = (int32_t)L->plans.size();
  L->plans.push_back(std::move(pl));
  return BBX_OK;
}

bbx_status bbx_loader_add_scalar(bbx_loader* L, int32_t field_index, int32_t* plan_id) {
  if (!L) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null loader");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "loader already started");
  const bbx_dataset* ds = L->ds;
  if (field_index < 0 || field_index >= (int)ds->fields.size() || ds->fields[field_index].info.kind > 1)
    return (bbx_status)fail(BBX_SCHEMA_MISMATCH, "field %d is not a scalar field", field_index);
  cudaSetDevice(L->device);
  Plan pl;
  pl.field_index = field_index;
  pl.scalar = true;
  pl.outs.assign(L->nslots, nullptr);
  // column upload once (Dataset.column, reader.py:391-406)
  std::vector<uint64_t> col((size_t)std::max<int64_t>(ds->num_samples, 1));
  for (int64_t i = 0; i < ds->num_samples; ++i) col[i] = bbx::u64_cell(ds, i, ds->fields[field_index]);
  cudaError_t e = cudaMalloc(&pl.d_col, col.size() * 8);
  if (e == cudaSuccess) e = cudaMemcpy(pl.d_col, col.data(), col.size() * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return (bbx_status)fail(BBX_CUDA_ERROR, "scalar column upload: %s", cudaGetErrorString(e));
  *plan_id = (int32_t)L->plans.size();
  L->plans.push_back(std::move(pl));
  return BBX_OK;
}

bbx_status bbx_loader_bind(bbx_loader* L, int32_t plan_id, int32_t slot, void* out_dev) {
  if (!L || plan_id < 0 || plan_id >= (int)L->plans.size() || slot < 0 || slot >= L->nslots)
    return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad plan or slot");
  L->plans[plan_id].outs[slot] = out_dev;
  return BBX_OK;
}

bbx_status bbx_loader_submit(bbx_loader* L, int32_t slot, const int64_t* idx, int32_t count, uint64_t seed,
                             uint64_t epoch) {
  if (!L || slot < 0 || slot >= L->nslots) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad slot");
  if (count < 0 || count > L->batch) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "count %d outside [0, %d]", count, L->batch);
  for (auto& pl : L->plans)
    if (!pl.outs[slot]) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "slot %d has unbound outputs", slot);
  int rc = bbx::finalize(L);
  if (rc) return (bbx_status)rc;
  std::lock_guard<std::mutex> g(L->mu);
  if (L->stop) return (bbx_status)fail(BBX_SHUTDOWN, "loader shut down");
  Slot& S = L->slots[slot];
  if (S.state == 1) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "slot %d already has a batch in flight", slot);
  S.idx.assign(idx, idx + count);
  S.count = count; S.seed = seed; S.epoch = epoch;
  S.state = 1; S.fatal = 0;
  L->queue.push_back(slot);
  L->cv.notify_one();
  return BBX_OK;
}

bbx_status bbx_loader_wait(bbx_loader* L, int32_t slot, int64_t* bad_pos) {
  if (!L || slot < 0 || slot >= L->nslots) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad slot");
  if (bad_pos) *bad_pos = -1;
  auto t0 = std::chrono::steady_clock::now();
  Slot& S = L->slots[slot];
  {
    std::unique_lock<std::mutex> lk(L->mu);
    if (S.state == 0) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "slot %d has no batch", slot);
    L->done_cv.wait(lk, [&] { return S.state == 2; });
  }
  cudaSetDevice(L->device);
  if (S.fatal) return (bbx_status)fail(S.fatal, "%s", S.fatal_msg.c_str());
  // The host waits for the batch's device work only when it has something to read
  // back: per-sample device status (RLE / JPEG) or a profiling window.  Otherwise the
  // batch is complete as far as the host knows (host-side sample errors are final),
  // and the consumer's stream is ordered after it by bbx_loader_stream_wait -- the
  // consumer keeps slot_count - 1 batches queued on the GPU instead of syncing per step.
  bool need_sync = false;
  for (size_t p = 0; p < L->plans.size(); ++p) need_sync = need_sync || S.plan_has_rle[p] || S.plan_has_jpeg[p];
  cudaError_t e = need_sync ? cudaEventSynchronize(S.done) : cudaSuccess;
  {
    std::lock_guard<std::mutex> g(L->stats_mu);
    L->stats.wait_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  if (e != cudaSuccess) return (bbx_status)fail(BBX_CUDA_ERROR, "batch failed on device: %s", cudaGetErrorString(e));
  // merge host-detected and device-detected per-sample failures: lowest position wins
  HostErr best = S.herr;
  for (size_t p = 0; p < L->plans.size(); ++p) {
    if (!S.plan_has_rle[p] && !S.plan_has_jpeg[p]) continue;
    const Plan& pl = L->plans[p];
    const uint8_t* dblk = S.h_stage + L->desc_off[p];
    for (int pos = 0; pos < S.count; ++pos) {
      if (best.pos >= 0 && (pos > best.pos || (pos == best.pos && (int)p >= best.plan))) break;
      const SampleDesc* d = reinterpret_cast<const SampleDesc*>(dblk + (size_t)pos * pl.dev.desc_stride);
      if (d->skip || (d->codec != CODEC_RLE && d->codec != CODEC_JPEG)) continue;
      if (d->codec == CODEC_RLE && !S.plan_has_rle[p]) continue;
      if (d->codec == CODEC_JPEG && !S.plan_has_jpeg[p]) continue;
      const SampleStatus& st = S.h_status[p * L->batch + pos];
      if (st.kind == 0) continue;
      char buf[256];
      int64_t n = (int64_t)d->h * d->w * d->c;
      if (st.kind == 1) std::snprintf(buf, sizeof buf, "rle runs sum past %lld bytes", (long long)n);
      else if (st.kind == 2) std::snprintf(buf, sizeof buf, "rle runs sum to %lld bytes, expected %lld", (long long)st.value, (long long)n);
      else std::snprintf(buf, sizeof buf, "jpeg: bad Huffman code in restart interval %lld", (long long)st.value);
      best.pos = pos; best.plan = (int)p; best.code = BBX_CORRUPT_PAYLOAD; best.msg = buf;
      break;
    }
  }
  if (best.pos >= 0) {
    if (bad_pos) *bad_pos = best.pos;
    return (bbx_status)fail(best.code, "%s", best.msg.c_str());
  }
  return BBX_OK;
}

bbx_status bbx_loader_stream_wait(bbx_loader* L, int32_t slot, void* stream) {
  if (!L || slot < 0 || slot >= L->nslots) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad slot");
  cudaSetDevice(L->device);
  cudaError_t e = cudaStreamWaitEvent((cudaStream_t)stream, L->slots[slot].done, 0);
  if (e != cudaSuccess) return (bbx_status)fail(BBX_CUDA_ERROR, "stream wait: %s", cudaGetErrorString(e));
  return BBX_OK;
}

bbx_status bbx_loader_step(bbx_loader* L, int32_t release_slot, int32_t submit_slot, const int64_t* idx,
                           int32_t count, uint64_t seed, uint64_t epoch, int32_t wait_slot, void* stream,
                           int64_t* bad_pos) {
  if (bad_pos) *bad_pos = -1;
  if (release_slot >= 0)
    if (bbx_status r = bbx_loader_release(L, release_slot, stream)) return r;
  if (submit_slot >= 0)
    if (bbx_status r = bbx_loader_submit(L, submit_slot, idx, count, seed, epoch)) return r;
  if (bbx_status r = bbx_loader_wait(L, wait_slot, bad_pos)) return r;
  return bbx_loader_stream_wait(L, wait_slot, stream);
}

bbx_status bbx_loader_release(bbx_loader* L, int32_t slot, void* stream) {
  if (!L || slot < 0 || slot >= L->nslots) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "bad slot");
  if (!L->finalized) return BBX_OK;
  cudaSetDevice(L->device);
  std::lock_guard<std::mutex> g(L->mu);
  Slot& S = L->slots[slot];
  cudaError_t e = cudaEventRecord(S.release, (cudaStream_t)stream);
  if (e != cudaSuccess) return (bbx_status)fail(BBX_CUDA_ERROR, "release record: %s", cudaGetErrorString(e));
  S.released_pending = true;
  if (S.state == 2) S.state = 0;
  return BBX_OK;
}

bbx_status bbx_loader_drain(bbx_loader* L) {
  if (!L) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null loader");
  if (!L->finalized) return BBX_OK;
  {
    std::unique_lock<std::mutex> lk(L->mu);
    L->done_cv.wait(lk, [&] {
      if (!L->queue.empty()) return false;
      for (auto& S : L->slots) if (S.state == 1) return false;
      return true;
    });
    for (auto& S : L->slots) if (S.state == 2) S.state = 0;
    L->pp.plans.clear();   // an abandoned stream's remaining page plan
  }
  cudaSetDevice(L->device);
  cudaError_t e1 = cudaStreamSynchronize(L->comp_st[0]), e2 = cudaStreamSynchronize(L->copy_st);
  if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(L->comp_st[1]);
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    return (bbx_status)fail(BBX_CUDA_ERROR, "drain: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  return BBX_OK;
}

void bbx_loader_destroy(bbx_loader* L) {
  if (!L) return;
  if (L->finalized) {
    bbx_loader_drain(L);
    { std::lock_guard<std::mutex> g(L->mu); L->stop = true; }
    L->cv.notify_all();
    if (L->th.joinable()) L->th.join();
  }
  cudaSetDevice(L->device);
  if (L->pp.d_pool) cudaFree(L->pp.d_pool);
  if (L->pp.h_buf) {
    cudaFreeHost(L->pp.h_buf);
    for (int k = 0; k < kPageBufs; ++k) cudaEventDestroy(L->pp.buf_ev[k]);
  }
  for (auto& S : L->slots) {
    if (S.h_stage) cudaFreeHost(S.h_stage);
    if (S.d_stage) cudaFree(S.d_stage);
    if (S.d_status) cudaFree(S.d_status);
    if (S.h_status) cudaFreeHost(S.h_status);
    if (&S == &L->slots[0] && L->t_ref) { cudaEventDestroy(L->t_ref); L->t_ref = nullptr; }
    for (int k = 0; k < kStreams; ++k)
      if (S.gexec[k]) cudaGraphExecDestroy(S.gexec[k]);
    if (S.h2d_done) cudaEventDestroy(S.h2d_done);
    if (S.h2d_t) cudaEventDestroy(S.h2d_t);
    if (S.done) cudaEventDestroy(S.done);
    if (S.release) cudaEventDestroy(S.release);
    if (S.k0) cudaEventDestroy(S.k0);
    if (S.k1) cudaEventDestroy(S.k1);
  }
  for (auto& pl : L->plans) {
    if (pl.d_lut) cudaFree(pl.d_lut);
    if (pl.d_col) cudaFree(pl.d_col);
    for (auto* p : pl.d_scratch) if (p) cudaFree(p);
    for (auto* p : pl.d_tables) if (p) cudaFree(p);
    for (int k = 0; k < kStreams; ++k) {
      if (pl.d_coef[k]) cudaFree(pl.d_coef[k]);
      if (pl.d_planes[k]) cudaFree(pl.d_planes[k]);
      if (pl.d_ticket[k]) cudaFree(pl.d_ticket[k]);
    }
  }
  if (L->jt.h_huff) cudaFreeHost(L->jt.h_huff);
  if (L->jt.h_quant) cudaFreeHost(L->jt.h_quant);
  if (L->jt.d_huff) cudaFree(L->jt.d_huff);
  if (L->jt.d_quant) cudaFree(L->jt.d_quant);
  if (L->copy_st) cudaStreamDestroy(L->copy_st);
  for (cudaStream_t st : L->comp_st) if (st) cudaStreamDestroy(st);
  delete L;
}

bbx_status bbx_loader_set_zero_copy(bbx_loader* L, int enabled) {
  if (!L) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null loader");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "loader already started");
  L->zero_copy = enabled != 0;
  return BBX_OK;
}

bbx_status bbx_loader_prefetch_headers(bbx_loader* L, const int64_t* idx, int64_t n) {
  if (!L || (n > 0 && !idx)) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "loader already started");
  L->prefetch_set.assign(idx, idx + std::max<int64_t>(n, 0));
  std::sort(L->prefetch_set.begin(), L->prefetch_set.end());   // distinct: one pool task per sample
  L->prefetch_set.erase(std::unique(L->prefetch_set.begin(), L->prefetch_set.end()), L->prefetch_set.end());
  return BBX_OK;
}

bbx_status bbx_loader_set_option(bbx_loader* L, const char* name, int64_t value) {
  if (!L || !name) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "loader already started");
  const std::string n(name);
  if (n == "window_staging") L->window_staging = value != 0;
  else if (n == "jpeg_header_cache") L->jpeg_cache = value != 0;
  else if (n == "jpeg_roi") L->jpeg_roi = value != 0;
  else if (n == "jpeg_header_prefetch") L->jpeg_prefetch = value != 0;
  else if (n == "direct_io") { L->direct_io = value != 0; if (L->direct_io) { L->window_staging = false; } }
  else if (n == "read_latency_ns") L->read_latency_ns = value > 0 ? value : 0;
  else if (n == "parallel_desc_min") L->par_desc_min = value;
  else if (n == "cuda_graphs") L->use_graphs = value != 0;
  else if (n == "zc_gather") L->zc_gather = value != 0;
  else if (n == "compute_streams") {
    if (value < 1 || value > kStreams) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "compute_streams must be 1 or %d", kStreams);
    L->nstreams = (int)value;
  }
  else return (bbx_status)fail(BBX_INVALID_ARGUMENT, "unknown loader option '%s'", name);
  return BBX_OK;
}

bbx_status bbx_loader_get_stats(const bbx_loader* L, bbx_loader_stats* out) {
  if (!L || !out) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  bbx_loader* M = const_cast<bbx_loader*>(L);
  std::lock_guard<std::mutex> g(M->stats_mu);
  if (L->finalized) {
    cudaSetDevice(L->device);
    for (auto& S : M->slots)   // profiled batches not yet read: wait for their windows
      if (S.timed && cudaEventSynchronize(S.k1) == cudaSuccess) collect_timing(M, S);
  }
  *out = L->stats;
  out->numa_node = L->numa_node;
  out->staging_threads = L->pool ? L->pool->size() : 0;
  out->staging_cpus = (int64_t)L->local_cpus.size();
  return BBX_OK;
}
bbx_status bbx_loader_reset_stats(bbx_loader* L) {
  if (!L) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null loader");
  std::lock_guard<std::mutex> g(L->stats_mu);
  L->stats = bbx_loader_stats{};
  for (auto& S : L->slots) S.timed = false;   // windows of batches before the reset are not counted
  L->last_k1_ms = -1.f;
  return BBX_OK;
}
bbx_status bbx_loader_set_profiling(bbx_loader* L, int enabled) {
  if (!L) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null loader");
  std::lock_guard<std::mutex> g(L->mu);
  L->profiling = enabled != 0;
  L->prof_every = enabled > 1 ? enabled : 1;
  L->prof_seq = 0;
  L->last_k1_ms = -1.f;
  return BBX_OK;
}
void* bbx_loader_compute_stream(bbx_loader* L) { return L ? (void*)L->comp_st[0] : nullptr; }

static int decode_image_impl(int32_t h, int32_t w, int32_t c, int32_t codec, const uint8_t* payload_host, int64_t len,
                             uint8_t* out_dev, int device) {
  // codecs.decode_image on device: a one-sample Decode plan with max dims (h, w).
  if (h < 1 || w < 1 || c < 1) return fail(BBX_SCHEMA_MISMATCH, "image dims must all be >= 1");
  int64_t n = (int64_t)h * w * c;
  if (codec == CODEC_RAW && len != n)
    return fail(BBX_CORRUPT_PAYLOAD, "raw payload is %lld bytes, expected %lld", (long long)len, (long long)n);
  if (codec == CODEC_RLE && len % 5) return fail(BBX_CORRUPT_PAYLOAD, "rle payload length is not a multiple of 5");
  if (codec == CODEC_SUB2) {
    int64_t m = (int64_t)((h + 1) / 2) * ((w + 1) / 2) * c;
    if (len != m) return fail(BBX_CORRUPT_PAYLOAD, "subsampled payload is %lld bytes, expected %lld", (long long)len, (long long)m);
  }
  if (codec == CODEC_JPEG) return jpeg_decode_one(h, w, c, payload_host, len, out_dev, device);
  if (codec < 0 || codec > 2) return fail(BBX_CORRUPT_PAYLOAD, "unknown codec %d", codec);
  CK(cudaSetDevice(device));
  PlanDev P{};
  P.src_kind = SRC_DECODE; P.canvas_h = h; P.canvas_w = w; P.channels = c; P.src_row_w = w;
  P.src_elem = 1; P.src_dtype = BBX_U8; P.out_h = h; P.out_w = w; P.out_c = c; P.out_dtype = BBX_U8;
  P.value_mode = VAL_COPY; P.desc_stride = kDescHeader + 8; P.rows_per_tile = std::min(16, h);
  for (;;) {
    P.lay = img_layout_host(P);
    P.smem_bytes = P.lay.total;
    if (P.smem_bytes <= kSmemBudget || P.rows_per_tile == 1) break;
    P.rows_per_tile /= 2;
  }
  if (P.smem_bytes > kSmemBudget || (int64_t)w * c + 64 > 65535) return fail(BBX_SPEC_MISMATCH, "image too wide");
  P.tiles_per_sample = (h + P.rows_per_tile - 1) / P.rows_per_tile;
  P.h_tpc = std::max(1, kThreads / w);
  P.tab_stride = image_tab_stride(P);
  P.scratch_bytes = (n + 15) / 16 * 16;
  P.out_sample_elems = n;
  if ((w + 3 * h) * 4 > kSmemBudget) return fail(BBX_SPEC_MISMATCH, "image too large");
  size_t dbytes = 64 + (size_t)((len + 15) / 16 * 16) + 64;
  uint8_t* d_buf = nullptr;
  uint8_t* d_scr = nullptr;
  uint32_t* d_tab = nullptr;
  SampleStatus* d_st = nullptr;
  CK(cudaMalloc(&d_buf, dbytes));
  CK(cudaMalloc(&d_tab, (size_t)P.tab_stride * 4 + 64));
  std::vector<uint8_t> hb(64, 0);
  SampleDesc* d = reinterpret_cast<SampleDesc*>(hb.data());
  d->src = 0; d->len = (uint32_t)len; d->h = (uint16_t)h; d->w = (uint16_t)w; d->c = (uint8_t)c; d->codec = (uint8_t)codec;
  cudaMemcpy(d_buf, hb.data(), 64, cudaMemcpyHostToDevice);
  if (len) cudaMemcpy(d_buf + 64, payload_host, (size_t)len, cudaMemcpyHostToDevice);
  cudaMalloc(&d_st, sizeof(SampleStatus));
  cudaMemset(d_st, 0, sizeof(SampleStatus));
  LaunchArgs A{};
  A.desc = d_buf; A.payload = d_buf + 64; A.out = out_dev; A.status = d_st; A.count = 1; A.tables = d_tab;
  int rc = 0;
  if (codec == CODEC_RLE) {
    cudaMalloc(&d_scr, P.scratch_bytes + 64);
    A.scratch = d_scr;
    rc |= launch_rle_expand(P, A, nullptr);
  }
  rc |= launch_image(P, A, nullptr);
  SampleStatus st{};
  cudaError_t e = cudaMemcpy(&st, d_st, sizeof st, cudaMemcpyDeviceToHost);
  cudaFree(d_buf); cudaFree(d_st); cudaFree(d_tab); if (d_scr) cudaFree(d_scr);
  if (rc || e != cudaSuccess) return fail(BBX_CUDA_ERROR, "decode failed: %s", cudaGetErrorString(e));
  if (st.kind == 1) return fail(BBX_CORRUPT_PAYLOAD, "rle runs sum past %lld bytes", (long long)n);
  if (st.kind == 2) return fail(BBX_CORRUPT_PAYLOAD, "rle runs sum to %lld bytes, expected %lld", (long long)st.value, (long long)n);
  return BBX_OK;
}

bbx_status bbx_decode_image(int32_t h, int32_t w, int32_t c, int32_t codec, const uint8_t* payload_host, int64_t len,
                            uint8_t* out_dev, int device) {
  return (bbx_status)decode_image_impl(h, w, c, codec, payload_host, len, out_dev, device);
}

static int set_page_pool_impl(bbx_loader* L, int64_t capacity_pages, double fetch_latency_s) {
  if (!L) return fail(BBX_INVALID_ARGUMENT, "null loader");
  if (L->finalized) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "page pool: set before the first submit");
  if (capacity_pages < 1)
    return (bbx_status)fail(BBX_CAPACITY_TOO_SMALL, "capacity_pages must be >= 1, got %lld", (long long)capacity_pages);
  if (L->ds->d_heap || L->zero_copy)
    return (bbx_status)fail(BBX_INVALID_ARGUMENT, "page pool: the heap is already device-resident / zero-copy");
  CK(cudaSetDevice(L->device));
  PagePool& PP = L->pp;
  PP.capacity = capacity_pages;
  PP.fetch_latency_s = fetch_latency_s > 0 ? fetch_latency_s : 0.0;
  const int64_t np = (L->ds->alloc_table_offset - L->ds->heap_offset) / L->ds->page_size;
  PP.slot_of.assign((size_t)std::max<int64_t>(np, 1), -1);
  if (!PP.h_buf) {
    CK(cudaHostAlloc(&PP.h_buf, (size_t)kPageBufs * L->ds->page_size, cudaHostAllocDefault));
    for (int k = 0; k < kPageBufs; ++k) CK(cudaEventCreateWithFlags(&PP.buf_ev[k], cudaEventDisableTiming));
  }
  return BBX_OK;
}
bbx_status bbx_loader_set_page_pool(bbx_loader* L, int64_t capacity_pages, double fetch_latency_s) {
  return (bbx_status)set_page_pool_impl(L, capacity_pages, fetch_latency_s);
}

bbx_status bbx_loader_plan_epoch(bbx_loader* L, const int64_t* idx, const int32_t* batch_len, int32_t n_batches,
                                 int64_t* planned_fetches, int64_t* planned_reloads) {
  if (!L || (n_batches > 0 && (!idx || !batch_len))) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "null argument");
  if (!L->pp.capacity) return (bbx_status)fail(BBX_INVALID_ARGUMENT, "page pool: not enabled");
  PagePlan P;
  if (int r = plan_epoch(L, idx, batch_len, n_batches, P)) return (bbx_status)r;
  if (planned_fetches) *planned_fetches = P.fetches;
  if (planned_reloads) *planned_reloads = P.reloads;
  if (n_batches > 0) {
    std::lock_guard<std::mutex> g(L->mu);
    L->pp.plans.push_back(std::move(P));
  }
  return BBX_OK;
}

bbx_status bbx_jpeg_check(int32_t h, int32_t w, int32_t c, const uint8_t* payload, int64_t len) {
  if (len < 4 || len > 0xFFFFFFFFll) return (bbx_status)fail(BBX_CORRUPT_PAYLOAD, "jpeg: missing SOI marker");
  if (h < 1 || w < 1 || h > 65535 || w > 65535 || c < 1 || c > 255)
    return (bbx_status)fail(BBX_SCHEMA_MISMATCH, "image dims out of range");
  bbx_loader L;                                  // only its table registry is used (no device work)
  std::vector<JHuff> hh(kJpegMaxHuff);
  std::vector<JQuant> hq(kJpegMaxQuant);
  L.jt.h_huff = hh.data(); L.jt.h_quant = hq.data();
  Plan pl;
  pl.jpeg_blocks_cap = (int64_t)c * (2 * ((h + 15) / 16)) * (2 * ((w + 15) / 16));
  pl.jpeg_int_cap = (int64_t)((h + 7) / 8) * ((w + 7) / 8);
  uint8_t desc[64] = {0};
  SampleDesc* d = reinterpret_cast<SampleDesc*>(desc);
  d->len = (uint32_t)len; d->h = (uint16_t)h; d->w = (uint16_t)w; d->c = (uint8_t)c; d->codec = CODEC_JPEG;
  JpegDesc J{};
  std::vector<uint32_t> starts;
  HostErr err;
  const bool ok = jpeg_prepare(&L, pl, payload, (uint32_t)len, d, &J, &starts, err, 0, 0);
  L.jt.h_huff = nullptr; L.jt.h_quant = nullptr;
  return ok ? BBX_OK : (bbx_status)fail(err.code, "%s", err.msg.c_str());
}

}  // extern "C"
