// wn_alloc.cu -- the device-memory cache of libwn.
//
// Every build and every query needs large temporary buffers (records, the
// query permutation, the hard-pair queue: ~1 GB for the C5 batch).  Mapping
// them anew on every call costs milliseconds of host time, so freed blocks are
// kept in a per-device cache and reused.  Stream safety: a freed block carries
// an event recorded on the stream that last used it; a later allocation on a
// different stream waits on that event (cudaStreamWaitEvent) before reuse, so
// reuse is stream-ordered exactly like cudaMallocAsync.
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "wn_common.cuh"

namespace wn {

namespace {
struct Block {
  void *p;
  size_t size;
  int dev;
  cudaStream_t st;
  cudaEvent_t ev;
};
std::mutex g_mu;
std::multimap<size_t, Block> g_free;             // by size
std::unordered_map<void *, Block> g_live;         // allocated blocks

size_t size_class(size_t b) {
  if (b < 512) return 512;
  if (b < (1u << 20)) {
    size_t s = 512;
    while (s < b) s <<= 1;
    return s;
  }
  const size_t g = (size_t)2 << 20;               // 2 MiB granules above 1 MiB
  return (b + g - 1) / g * g;
}
}  // namespace

// WN_ALLOC_EXACT=1 (sanitizer runs): every block is a fresh cudaMalloc of the
// exact size, freed with cudaFree -- no size-class slack and no reuse, so
// compute-sanitizer's memcheck sees every out-of-bounds access.
static bool alloc_exact() {
  static const int v = [] { const char *s = std::getenv("WN_ALLOC_EXACT"); return (s && *s && *s != '0') ? 1 : 0; }();
  return v != 0;
}

// WN_ALLOC_POISON=1 (checked runs): every block handed out is first filled
// with 0xA5 bytes (NaN-like doubles, huge ints), so a kernel that reads memory
// nobody wrote changes its results -- the determinism / parity comparisons of
// scripts/checked_run.sh then catch it (an initcheck substitute).
static bool alloc_poison() {
  static const int v = [] { const char *s = std::getenv("WN_ALLOC_POISON"); return (s && *s && *s != '0') ? 1 : 0; }();
  return v != 0;
}
static cudaError_t cache_alloc_raw(void **out, size_t bytes, cudaStream_t st);

cudaError_t cache_alloc(void **out, size_t bytes, cudaStream_t st) {
  cudaError_t e = cache_alloc_raw(out, bytes, st);
  if (e == cudaSuccess && alloc_poison() && bytes) e = cudaMemsetAsync(*out, 0xA5, bytes, st);
  return e;
}

static cudaError_t cache_alloc_raw(void **out, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (alloc_exact()) return cudaMalloc(out, bytes ? bytes : 1);
  const size_t sz = size_class(bytes ? bytes : 1);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_free.lower_bound(sz); it != g_free.end() && it->first <= 2 * sz; ++it) {
      if (it->second.dev != dev) continue;
      Block b = it->second;
      g_free.erase(it);
      if (b.ev && b.st != st) {
        e = cudaStreamWaitEvent(st, b.ev, 0);
        if (e != cudaSuccess) return e;
      }
      b.st = st;
      g_live[b.p] = b;
      *out = b.p;
      return cudaSuccess;
    }
  }
  void *p = nullptr;
  e = cudaMalloc(&p, sz);
  if (e != cudaSuccess) {
    // retry once after dropping the cache
    cudaGetLastError();
    cache_trim();
    e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) return e;
  }
  Block b{p, sz, dev, st, nullptr};
  std::lock_guard<std::mutex> lk(g_mu);
  g_live[p] = b;
  *out = p;
  return cudaSuccess;
}

void cache_free(void *p, cudaStream_t st) {
  if (!p) return;
  if (alloc_exact()) {
    cudaStreamSynchronize(st);
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_live.find(p);
  if (it == g_live.end()) return;
  Block b = it->second;
  g_live.erase(it);
  if (!b.ev) cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
  b.st = st;
  if (b.ev) cudaEventRecord(b.ev, st);
  g_free.emplace(b.size, b);
}

void cache_trim() {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto &kv : g_free) {
    if (kv.second.ev) {
      cudaEventSynchronize(kv.second.ev);
      cudaEventDestroy(kv.second.ev);
    }
    cudaFree(kv.second.p);
  }
  g_free.clear();
}

}  // namespace wn

extern "C" void wn_trim_memory(void) { wn::cache_trim(); }
