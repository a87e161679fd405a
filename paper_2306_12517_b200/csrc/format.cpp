// .bbox container read side: mmap + header decode + row cells.
// Restates format.py:57-75 (layout), 298-337 (decode_header), 218-239
// (DatasetHeader.check), 147-162 (FieldDescriptor.check) and
// reader.py:323-366 (Dataset open, OsCache strategy).
#include "engine.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <set>

namespace bbx {

static uint16_t rd16(const uint8_t* p) { uint16_t v; std::memcpy(&v, p, 2); return v; }
static uint32_t rd32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
static uint64_t rd64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }

static int cell_width(int kind) {                      // format.py:94-100
  switch (kind) { case 0: case 1: case 2: return 8; case 3: return 16; case 4: return 24; }
  return -1;
}
static const int kArrayItem[4] = {1, 8, 4, 8};         // format.py:86-91

static std::string py_bytes_repr(const uint8_t* p, int n) {
  std::string s = "b'";
  char buf[8];
  for (int i = 0; i < n; ++i) {
    uint8_t c = p[i];
    if (c == '\\' || c == '\'') { s += '\\'; s += (char)c; }
    else if (c >= 32 && c < 127) s += (char)c;
    else { std::snprintf(buf, sizeof buf, "\\x%02x", c); s += buf; }
  }
  return s + "'";
}

int dataset_open(const char* path, bbx_dataset** out) {
  *out = nullptr;
  int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return fail(BBX_INVALID_FILE, "%s: cannot open: %s", path, std::strerror(errno));
  struct stat stt;
  if (fstat(fd, &stt) != 0) { ::close(fd); return fail(BBX_INVALID_FILE, "%s: stat failed", path); }
  size_t len = (size_t)stt.st_size;
  if (len < 56) { ::close(fd); return fail(BBX_INVALID_FILE, "%s: file shorter than header prefix", path); }
  void* m = mmap(nullptr, len, PROT_READ, MAP_SHARED, fd, 0);
  if (m == MAP_FAILED) { ::close(fd); return fail(BBX_INVALID_FILE, "%s: mmap failed", path); }
  madvise(m, len, MADV_WILLNEED);
  auto ds = std::make_unique<bbx_dataset>();
  ds->path = path; ds->fd = fd; ds->map = (const uint8_t*)m; ds->map_len = len;
  const uint8_t* b = ds->map;

  // HEADER_PREFIX "<8sIQHQQQQ2x"
  if (std::memcmp(b, "FASTDS01", 8) != 0) return fail(BBX_BAD_MAGIC, "bad magic %s", py_bytes_repr(b, 8).c_str());
  uint32_t version = rd32(b + 8);
  if (version != 1) return fail(BBX_UNSUPPORTED_VERSION, "unsupported version %u", version);
  ds->num_samples = (int64_t)rd64(b + 12);
  int nf = rd16(b + 20);
  ds->page_size = (int64_t)rd64(b + 22);
  ds->data_table_offset = (int64_t)rd64(b + 30);
  ds->heap_offset = (int64_t)rd64(b + 38);
  ds->alloc_table_offset = (int64_t)rd64(b + 46);
  size_t total = 56 + (size_t)124 * nf;
  if (len < total) return fail(BBX_INVALID_HEADER, "buffer too short for %d descriptors", nf);
  int off = 0;
  for (int i = 0; i < nf; ++i) {                       // DESCRIPTOR "<64sB48sI7x"
    const uint8_t* d = b + 56 + (size_t)124 * i;
    Field f{};
    int nlen = 0;
    while (nlen < 64 && d[nlen]) ++nlen;
    std::memcpy(f.info.name, d, nlen);
    f.info.name[nlen] = 0;
    int kind = d[64];
    if (kind > 4) return fail(BBX_INVALID_HEADER, "unknown field kind %d", kind);
    f.info.kind = kind;
    const uint8_t* prm = d + 65;
    if (kind == 2) {                                   // ARRAY_PARAMS "<BB2x4I"
      int code = prm[0], nd = prm[1];
      if (code > 3) return fail(BBX_INVALID_HEADER, "unknown array dtype code %d", code);
      if (nd < 1 || nd > 4) return fail(BBX_INVALID_HEADER, "array ndims out of range: %d", nd);
      f.info.array_dtype = code; f.info.ndims = nd;
      int64_t nbytes = kArrayItem[code];
      for (int k = 0; k < nd; ++k) { f.info.dims[k] = rd32(prm + 4 + 4 * k); nbytes *= f.info.dims[k]; }
      f.array_nbytes = nbytes;
    } else if (kind == 4) {                            // IMAGE_PARAMS "<HHB"
      f.info.max_height = rd16(prm); f.info.max_width = rd16(prm + 2); f.info.channels = prm[4];
    }
    uint32_t cw = rd32(d + 113);
    if ((int)cw != cell_width(kind))
      return fail(BBX_INVALID_HEADER, "field '%s': stored cell width %u != %d", f.info.name, cw, cell_width(kind));
    f.info.cell_offset = off;
    f.cell_width = (int)cw;
    off += (int)cw;
    ds->fields.push_back(f);
  }
  ds->row_width = off;
  // DatasetHeader.check (format.py:218-239)
  if (nf == 0) return fail(BBX_INVALID_HEADER, "at least one field is required");
  std::set<std::string> names;
  for (auto& f : ds->fields) {
    size_t nl = std::strlen(f.info.name);
    if (nl == 0 || nl > 63) return fail(BBX_INVALID_HEADER, "field name must be 1..63 bytes: '%s'", f.info.name);
    if (!names.insert(f.info.name).second) return fail(BBX_INVALID_HEADER, "field names must be unique");
    if (f.info.kind == 2)
      for (int k = 0; k < f.info.ndims; ++k)
        if (f.info.dims[k] < 1) return fail(BBX_INVALID_HEADER, "array dims must be positive u32 values");
    if (f.info.kind == 4) {
      if (f.info.max_height < 1 || f.info.max_width < 1) return fail(BBX_INVALID_HEADER, "image max dims must be in 1..65535");
      if (f.info.channels < 1) return fail(BBX_INVALID_HEADER, "image channels must be in 1..255");
    }
  }
  if (ds->page_size < 65536 || (ds->page_size & (ds->page_size - 1)))
    return fail(BBX_INVALID_HEADER, "page_size must be a power of two >= 65536");
  if (ds->data_table_offset != (int64_t)total) return fail(BBX_INVALID_HEADER, "data_table_offset must equal the header byte length");
  if (ds->heap_offset % ds->page_size) return fail(BBX_INVALID_HEADER, "heap_offset must be page aligned");
  if (!(ds->data_table_offset < ds->heap_offset && ds->heap_offset <= ds->alloc_table_offset))
    return fail(BBX_INVALID_HEADER, "sections must be ordered header < heap <= alloc table");
  if ((uint64_t)ds->num_samples > (uint64_t)1 << 40 ||
      ds->data_table_offset + ds->num_samples * ds->row_width > (int64_t)len)
    return fail(BBX_INVALID_FILE, "%s: data table truncated", path);
  if (ds->alloc_table_offset > (int64_t)len) return fail(BBX_INVALID_FILE, "%s: heap truncated", path);
  ds->rows = b + ds->data_table_offset;
  *out = ds.release();
  return BBX_OK;
}

void dataset_close(bbx_dataset* ds) {
  if (!ds) return;
  if (ds->d_heap) { cudaSetDevice(ds->resident_device); cudaFree(ds->d_heap); }
  if (ds->h_heap) cudaFreeHost(ds->h_heap);
  delete ds;   // ~bbx_dataset unmaps and closes
}

ImageCell image_cell(const bbx_dataset* ds, int64_t i, const Field& f) {   // "<QQHHBB2x"
  const uint8_t* p = ds->rows + i * ds->row_width + f.info.cell_offset;
  ImageCell c;
  c.offset = rd64(p); c.length = rd64(p + 8); c.h = rd16(p + 16); c.w = rd16(p + 18); c.c = p[20]; c.codec = p[21];
  return c;
}
uint64_t u64_cell(const bbx_dataset* ds, int64_t i, const Field& f) {
  return rd64(ds->rows + i * ds->row_width + f.info.cell_offset);
}

int64_t primary_page(const bbx_dataset* ds, int64_t i) {           // reader.py:430-437
  for (auto& f : ds->fields) {
    if (f.info.kind == 2) return ((int64_t)u64_cell(ds, i, f) - ds->heap_offset) / ds->page_size;
    if (f.info.kind == 3 || f.info.kind == 4) {
      const uint8_t* p = ds->rows + i * ds->row_width + f.info.cell_offset;
      uint64_t o = rd64(p), l = rd64(p + 8);
      if (l) return ((int64_t)o - ds->heap_offset) / ds->page_size;
    }
  }
  return -1;
}

// Pinned host copy of the heap: the page cache's bytes held page-locked so the
// copy engine can DMA batch payloads without a CPU gather.
int dataset_pin_host(bbx_dataset* ds, int threads) {
  if (ds->h_heap) return BBX_OK;
  size_t heap = (size_t)(ds->alloc_table_offset - ds->heap_offset);
  uint8_t* h = nullptr;
  CK(cudaHostAlloc(&h, heap + 256, cudaHostAllocPortable | cudaHostAllocMapped));
  std::memset(h + heap, 0, 256);
  const size_t chunk = 64ull << 20;
  const size_t nchunks = (heap + chunk - 1) / chunk;
  threads = std::max(1, std::min(threads, (int)std::max<size_t>(nchunks, 1)));
  std::vector<std::thread> th;
  std::atomic<size_t> next{0};
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&] {
      for (size_t k; (k = next.fetch_add(1)) < nchunks;) {
        size_t o = k * chunk, n = std::min(chunk, heap - o);
        std::memcpy(h + o, ds->map + ds->heap_offset + o, n);
      }
    });
  for (auto& t : th) t.join();
  ds->h_heap = h;
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, h, 0) == cudaSuccess) ds->h_heap_dev = static_cast<uint8_t*>(dp);
  else cudaGetLastError();
  return BBX_OK;
}

int dataset_make_resident(bbx_dataset* ds, int device) {
  if (ds->d_heap) return BBX_OK;
  CK(cudaSetDevice(device));
  size_t heap = (size_t)(ds->alloc_table_offset - ds->heap_offset);
  uint8_t* d = nullptr;
  CK(cudaMalloc(&d, heap + 256));
  CK(cudaMemset(d + heap, 0, 256));
  // chunked copy through a pinned bounce buffer (the mmap is pageable)
  const size_t chunk = 64 << 20;
  uint8_t* bounce[2] = {nullptr, nullptr};
  cudaEvent_t ev[2];
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) { CK(cudaHostAlloc(&bounce[k], chunk, cudaHostAllocDefault)); CK(cudaEventCreate(&ev[k])); }
  int k = 0;
  for (size_t o = 0; o < heap; o += chunk, k ^= 1) {
    size_t n = std::min(chunk, heap - o);
    CK(cudaEventSynchronize(ev[k]));
    std::memcpy(bounce[k], ds->map + ds->heap_offset + o, n);
    CK(cudaMemcpyAsync(d + o, bounce[k], n, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(ev[k], st));
  }
  CK(cudaStreamSynchronize(st));
  for (int j = 0; j < 2; ++j) { cudaFreeHost(bounce[j]); cudaEventDestroy(ev[j]); }
  cudaStreamDestroy(st);
  ds->d_heap = d;
  ds->resident_device = device;
  return BBX_OK;
}

}  // namespace bbx
