// Workspace caching allocator and pinned small reads (common.cuh).
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace spb {

namespace {

static size_t env_size(const char* name, size_t dflt, int shift) {
  const char* e = std::getenv(name);
  return e ? (size_t)std::strtoull(e, nullptr, 10) << shift : dflt;
}
// Every block size is cached, up to 64 GB per device (SPB_WS_CACHE_MAX_MB: largest
// cached block, SPB_WS_CACHE_CAP_GB: cached bytes per device).  Until the last
// session of round 2 blocks above 256 MB went back to the CUDA mempool; a
// cudaMallocAsync of a multi-GB block from that pool (release threshold
// UINT64_MAX, nothing handed back to the driver) still stalled the host for
// 8 ms - 2 s in about every third cfg5 power_id call (CUPTI timeline,
// scripts/id_spread.py: kernel time 470 ms in every call, device span 502 -
// 2882 ms; with the blocks kept here 472 - 506 ms).  The footprint between
// calls is the same as before (the pool kept the memory too);
// sp_release_workspaces() hands both back.
const size_t kWsCacheMax = env_size("SPB_WS_CACHE_MAX_MB", size_t(64) << 30, 20);
const size_t kWsCacheCap = env_size("SPB_WS_CACHE_CAP_GB", size_t(64) << 30, 30);

// 512-byte granules up to 64 KB, then 8 steps per power of two (<= 12.5 % slack)
size_t ws_round(size_t b) {
  if (b <= 65536) return (b + 511) & ~size_t(511);
  int e = 63 - __builtin_clzll(b);
  size_t step = size_t(1) << (e - 3);
  return (b + step - 1) & ~(step - 1);
}

struct DevCache {
  std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free;
  size_t cached = 0;
  bool pool_tuned = false;
};

std::mutex g_mu;
DevCache g_dev[64];

DevCache* dev_cache() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
  DevCache* c = &g_dev[d];
  if (!c->pool_tuned) {
    // keep freed memory in the device's default pool across synchronisations
    // (a release threshold of 0 hands it back to the driver at every sync)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    c->pool_tuned = true;
  }
  return c;
}

void drain(DevCache* c) {
  for (auto& kv : c->free)
    for (void* p : kv.second) cudaFreeAsync(p, kv.first.first);
  c->free.clear();
  c->cached = 0;
}

}  // namespace

void* ws_alloc(size_t bytes, cudaStream_t s) {
  const size_t rb = ws_round(bytes);
  std::lock_guard<std::mutex> lk(g_mu);
  DevCache* c = dev_cache();
  if (!c) return nullptr;
  if (rb <= kWsCacheMax) {
    auto it = c->free.find({s, rb});
    if (it != c->free.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      c->cached -= rb;
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, rb, s) == cudaSuccess) return p;
  cudaGetLastError();
  // out of memory: hand every cached block back (and the pool's reserve to
  // the driver) and retry once
  if (std::getenv("SPB_HOST_TRACE")) std::fprintf(stderr, "spb ws_alloc: OOM on %zu bytes, draining\n", rb);
  drain(c);
  cudaDeviceSynchronize();
  {
    int d = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&d) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
  }
  if (cudaMallocAsync(&p, rb, s) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

void ws_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  const size_t rb = ws_round(bytes);
  std::lock_guard<std::mutex> lk(g_mu);
  DevCache* c = dev_cache();
  if (c && rb <= kWsCacheMax && c->cached + rb <= kWsCacheCap) {
    c->free[{s, rb}].push_back(p);
    c->cached += rb;
    return;
  }
  cudaFreeAsync(p, s);
}

void ws_release_all() {
  std::lock_guard<std::mutex> lk(g_mu);
  DevCache* c = dev_cache();
  if (!c) return;
  drain(c);
  cudaDeviceSynchronize();
}

// ------------------------------------------------------------ pinned reads ----
namespace {
struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};
thread_local PinnedBuf t_pinned;
}  // namespace

int PinnedReads::add(void* host_dst, const void* dev_src, size_t bytes) {
  const size_t off = (used_ + 15) & ~size_t(15);
  if (n_ >= kMax || off + bytes > (size_t(64) << 10)) {
    set_error("PinnedReads: too many / too large small reads");
    return SP_ECUDA;
  }
  if (!t_pinned.p) {
    SPB_CUDA(cudaMallocHost(&t_pinned.p, size_t(64) << 10));
    t_pinned.cap = size_t(64) << 10;
  }
  SPB_CUDA(cudaMemcpyAsync(static_cast<char*>(t_pinned.p) + off, dev_src, bytes, cudaMemcpyDeviceToHost, s_));
  dst_[n_] = host_dst;
  off_[n_] = off;
  len_[n_++] = bytes;
  used_ = off + bytes;
  return SP_OK;
}

int PinnedReads::sync() {
  SPB_CUDA(cudaStreamSynchronize(s_));
  for (int i = 0; i < n_; ++i) std::memcpy(dst_[i], static_cast<char*>(t_pinned.p) + off_[i], len_[i]);
  n_ = 0;
  used_ = 0;
  return SP_OK;
}

int read_small(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t s) {
  PinnedReads r(s);
  SPB_TRY(r.add(host_dst, dev_src, bytes));
  return r.sync();
}

// ------------------------------------------------------------ host trace ----
namespace {
struct HostTrace {
  std::vector<std::pair<const char*, double>> ev;
};
thread_local HostTrace t_trace;
const bool g_trace_on = std::getenv("SPB_HOST_TRACE") != nullptr;
}  // namespace

void host_mark(const char* tag) {
  if (!g_trace_on) return;
  const double us = std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count();
  t_trace.ev.emplace_back(tag, us);
}

std::string host_trace_dump() {
  std::string out;
  char buf[160];
  for (size_t i = 0; i < t_trace.ev.size(); ++i) {
    const double d = i ? t_trace.ev[i].second - t_trace.ev[i - 1].second : 0.0;
    std::snprintf(buf, sizeof(buf), "%9.1f %+8.1f  %s\n", t_trace.ev[i].second - t_trace.ev[0].second, d,
                  t_trace.ev[i].first);
    out += buf;
  }
  t_trace.ev.clear();
  return out;
}

}  // namespace spb
