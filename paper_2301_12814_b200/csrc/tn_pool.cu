// Device memory pool for plan tables and staging workspaces (include/tn_theta.h,
// tn_release_cached_memory). A simulation builds one plan per gate (new bond charges each time), so
// the plan's device memory is recycled instead of cudaMalloc/cudaFree per gate (cudaFree also
// synchronises the device). Reuse is stream-safe: a released block carries an event recorded on the
// stream of the last exec that used it, and is only handed out again once that event has completed.
#include <mutex>

#include "tn_internal.cuh"

namespace tn {
namespace {

struct Block {
  void* ptr = nullptr;
  size_t bytes = 0;
  int dev = 0;
  cudaEvent_t ev = nullptr;  // completion of the last work that used the block (nullptr: none)
  bool in_use = false;
};

std::mutex g_mu;
std::vector<Block> g_blocks;

size_t round_bytes(size_t b) {
  const size_t g = b >= (size_t(1) << 24) ? (size_t(2) << 20) : 4096;
  return (b + g - 1) / g * g;
}

bool ready(Block& b) {
  if (!b.ev) return true;
  cudaError_t e = cudaEventQuery(b.ev);
  if (e == cudaSuccess) return true;
  if (e != cudaErrorNotReady) cudaGetLastError();
  return false;
}

size_t free_idle_locked(bool wait) {
  size_t freed = 0;
  for (size_t i = 0; i < g_blocks.size();) {
    Block& b = g_blocks[i];
    if (!b.in_use && (wait || ready(b))) {
      if (b.ev) {
        cudaEventSynchronize(b.ev);
        cudaEventDestroy(b.ev);
      }
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != b.dev) cudaSetDevice(b.dev);
      cudaFree(b.ptr);
      if (cur != b.dev) cudaSetDevice(cur);
      freed += b.bytes;
      g_blocks[i] = g_blocks.back();
      g_blocks.pop_back();
    } else {
      ++i;
    }
  }
  return freed;
}

}  // namespace

void* pool_alloc(size_t bytes, cudaError_t* err) {
  *err = cudaSuccess;
  if (bytes == 0) return nullptr;
  bytes = round_bytes(bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  int best = -1;
  for (int i = 0; i < (int)g_blocks.size(); ++i) {
    Block& b = g_blocks[i];
    if (b.in_use || b.dev != dev || b.bytes < bytes || b.bytes > 2 * bytes + (size_t(2) << 20)) continue;
    if (!ready(b)) continue;
    if (best < 0 || b.bytes < g_blocks[best].bytes) best = i;
  }
  if (best >= 0) {
    g_blocks[best].in_use = true;
    return g_blocks[best].ptr;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    free_idle_locked(true);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    *err = e;
    return nullptr;
  }
  Block b;
  b.ptr = p;
  b.bytes = bytes;
  b.dev = dev;
  b.in_use = true;
  g_blocks.push_back(b);
  return p;
}

void pool_release(void* ptr, cudaStream_t last_stream, bool used) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_mu);
  for (Block& b : g_blocks) {
    if (b.ptr != ptr) continue;
    b.in_use = false;
    if (used) {
      if (!b.ev) cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
      if (b.ev && cudaEventRecord(b.ev, last_stream) != cudaSuccess) {
        cudaGetLastError();
        cudaDeviceSynchronize();  // cannot track the stream: make the block safe the slow way
      }
    }
    return;
  }
}

}  // namespace tn

extern "C" TN_API tn_status tn_release_cached_memory(int64_t* freed, int64_t* cached) {
  std::lock_guard<std::mutex> lk(tn::g_mu);
  const size_t f = tn::free_idle_locked(true);
  size_t held = 0;
  for (const auto& b : tn::g_blocks) held += b.bytes;
  if (freed) *freed = (int64_t)f;
  if (cached) *cached = (int64_t)held;
  return TN_OK;
}
