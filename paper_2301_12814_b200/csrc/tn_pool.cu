// Device memory pool for plan tables and staging workspaces (include/tn_theta.h,
// tn_release_cached_memory). A simulation builds one plan per gate (new bond charges each time), so
// the plan's device memory is recycled instead of cudaMalloc/cudaFree per gate (cudaFree also
// synchronises the device). Reuse is stream-safe: a released block carries an event recorded on the
// stream of the last exec that used it, and is only handed out again once that event has completed.
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>

#include "tn_internal.cuh"

namespace tn {
namespace {

struct Block {
  void* ptr = nullptr;
  size_t bytes = 0;
  int dev = 0;
  cudaEvent_t ev = nullptr;  // completion of the last work that used the block (nullptr: none)
  Fence* fence = nullptr;    // or a shared fence (a destroyed plan's last-use event, pool_release_fenced)
  bool in_use = false;
  uint64_t stamp = 0;        // release order (backpressure waits on the earliest)
  size_t req = 0;            // bytes last requested for it (tn_plan_reserve reserves blocks that fit this)
};
uint64_t g_stamp = 0;

std::mutex g_mu;
std::vector<Block> g_blocks;

size_t round_bytes(size_t b) {
  const size_t g = b >= (size_t(1) << 24) ? (size_t(2) << 20) : 4096;
  return (b + g - 1) / g * g;
}

// size of a NEW block: large requests round up to 1/16 of their power-of-two octave (≤ 6.25% slack) so that
// plans of slightly different shape (the ranks of a row sharding, successive gates of a sweep) share blocks
size_t grow_bytes(size_t b) {
  if (b < (size_t(1) << 24)) return b;
  size_t o = size_t(1) << 24;
  while (o * 2 <= b) o *= 2;
  const size_t g = o / 16;
  return (b + g - 1) / g * g;
}

bool fits(const Block& b, size_t bytes, int dev) {
  return b.dev == dev && b.bytes >= bytes && b.bytes <= 2 * bytes + (size_t(2) << 20);
}

void drop_fence(Block& b) {
  if (b.fence && --b.fence->refs == 0) {
    cudaEventDestroy(b.fence->ev);
    delete b.fence;
  }
  b.fence = nullptr;
}

bool ready(Block& b) {
  cudaEvent_t ev = b.fence ? b.fence->ev : b.ev;
  if (!ev) return true;
  cudaError_t e = cudaEventQuery(ev);
  if (e == cudaSuccess) {
    drop_fence(b);
    return true;
  }
  if (e != cudaErrorNotReady) cudaGetLastError();
  return false;
}

size_t free_idle_locked(bool wait) {
  size_t freed = 0;
  for (size_t i = 0; i < g_blocks.size();) {
    Block& b = g_blocks[i];
    if (!b.in_use && (wait || ready(b))) {
      if (b.fence) cudaEventSynchronize(b.fence->ev);
      drop_fence(b);
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
    if (b.in_use || !fits(b, bytes, dev)) continue;
    if (!ready(b)) continue;
    if (best < 0 || b.bytes < g_blocks[best].bytes) best = i;
  }
  if (best >= 0) {
    g_blocks[best].in_use = true;
    g_blocks[best].req = bytes;
    return g_blocks[best].ptr;
  }
  // Backpressure: a fitting block whose last use is still in flight is waited for rather than allocating
  // another one — a host that plans gates faster than the GPU runs them would otherwise grow the pool without
  // bound (and pay a cudaMalloc per gate); the earliest-released candidate completes first.
  int wait = -1;
  for (int i = 0; i < (int)g_blocks.size(); ++i) {
    Block& b = g_blocks[i];
    if (b.in_use || !fits(b, bytes, dev)) continue;
    if (wait < 0 || b.stamp < g_blocks[wait].stamp) wait = i;
  }
  if (wait >= 0) {
    Block& b = g_blocks[wait];
    cudaEvent_t ev = b.fence ? b.fence->ev : b.ev;
    if (ev && cudaEventSynchronize(ev) == cudaSuccess) {
      drop_fence(b);
      b.in_use = true;
      b.req = bytes;
      return b.ptr;
    }
    cudaGetLastError();
  }
  void* p = nullptr;
  size_t nb = grow_bytes(bytes);
  cudaError_t e = cudaMalloc(&p, nb);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    free_idle_locked(true);
    nb = bytes;
    e = cudaMalloc(&p, nb);
  }
  if (e != cudaSuccess) {
    *err = e;
    return nullptr;
  }
  Block b;
  b.ptr = p;
  b.bytes = nb;
  b.dev = dev;
  b.in_use = true;
  b.req = bytes;
  g_blocks.push_back(b);
  return p;
}

// tn_plan_reserve: at least `count` blocks (in use or idle) that a request like the one that produced `ptr`
// would accept; the missing ones are allocated now, idle
cudaError_t pool_reserve_like(const void* ptr, int count) {
  if (!ptr || count <= 0) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_mu);
  size_t req = 0;
  int dev = 0;
  for (const Block& b : g_blocks)
    if (b.ptr == ptr) {
      req = b.req;
      dev = b.dev;
    }
  if (req == 0) return cudaSuccess;
  int have = 0;
  for (const Block& b : g_blocks) have += fits(b, req, dev) ? 1 : 0;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaError_t e = cudaSuccess;
  for (; have < count; ++have) {
    Block b;
    b.bytes = grow_bytes(req);
    if ((e = cudaMalloc(&b.ptr, b.bytes)) != cudaSuccess) break;
    b.dev = dev;
    b.req = req;
    b.stamp = ++g_stamp;
    g_blocks.push_back(b);
  }
  if (cur != dev) cudaSetDevice(cur);
  return e;
}

Fence* fence_adopt(cudaEvent_t ev) {
  if (!ev) return nullptr;
  Fence* f = new (std::nothrow) Fence{ev, 0};
  if (!f) {  // cannot track it: make the event's work complete the slow way
    cudaEventSynchronize(ev);
    cudaEventDestroy(ev);
  }
  return f;
}

void pool_release_fenced(void* ptr, Fence* f) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_mu);
  for (Block& b : g_blocks) {
    if (b.ptr != ptr) continue;
    b.in_use = false;
    b.stamp = ++g_stamp;
    drop_fence(b);
    if (f) {
      b.fence = f;
      ++f->refs;
    }
    return;
  }
}

void fence_release(Fence* f) {  // a fence no block adopted
  if (f && f->refs == 0) {
    cudaEventDestroy(f->ev);
    delete f;
  }
}

void pool_release(void* ptr, cudaStream_t last_stream, bool used) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_mu);
  for (Block& b : g_blocks) {
    if (b.ptr != ptr) continue;
    b.in_use = false;
    b.stamp = ++g_stamp;
    drop_fence(b);
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

namespace {
std::mutex g_shell_mu;
std::vector<PlanShell> g_shells;
}  // namespace

cudaError_t shell_acquire(PlanShell* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_shell_mu);
    for (size_t i = 0; i < g_shells.size(); ++i)
      if (g_shells[i].dev == dev) {
        *out = g_shells[i];
        g_shells[i] = g_shells.back();
        g_shells.pop_back();
        return cudaSuccess;
      }
  }
  PlanShell sh;
  sh.dev = dev;
  if ((e = cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking)) != cudaSuccess) return e;
  for (auto& ev : sh.ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&sh.ev_ready, cudaEventDisableTiming)) != cudaSuccess) return e;
  *out = sh;
  return cudaSuccess;
}

// ---- pinned upload ring ----
// One process-wide pinned buffer, allocated once (never freed on the hot path: cudaFreeHost synchronises the
// device, and per-shell arenas that grew with the tables drained pipelined gates of MPO plans by 25%). Ranges are
// handed out FIFO; a range returns once the event of the plan that staged it has completed. Only small copies are
// staged — the fixed cost of a pageable cudaMemcpyAsync is what staging saves, while for a large table the host
// memcpy into the ring costs as much as the driver's own staging (MPO pair config 5: 7.2–7.5 ms per gate with
// every table staged vs 6.8–7.0 pageable); a full ring whose oldest range belongs to a plan still being built
// also falls back to pageable.
namespace {
constexpr size_t RING_BYTES = size_t(16) << 20;
constexpr size_t STAGE_MAX = size_t(256) << 10;
struct RingEvent {
  cudaEvent_t ev = nullptr;
  int refs = 0;
};
struct RingSeg {
  size_t start, end;
  const tn_plan* owner;
  RingEvent* done;        // nullptr until the owner seals
  bool complete = false;  // sealed without an event (its uploads were waited for on the host)
};
struct PinnedRing {
  std::mutex mu;
  char* base = nullptr;
  bool tried = false;
  size_t head = 0;
  std::deque<RingSeg> segs;
  std::vector<RingEvent*> free_ev;
};
PinnedRing& ring() {
  static PinnedRing r;
  return r;
}
void ring_pop_front(PinnedRing& r) {
  RingEvent* d = r.segs.front().done;
  r.segs.pop_front();
  if (d && --d->refs == 0) r.free_ev.push_back(d);
}
// reclaims completed ranges from the front; wait = block on the oldest sealed one
bool ring_reclaim(PinnedRing& r, bool wait) {
  bool any = false;
  while (!r.segs.empty()) {
    if (r.segs.front().complete) {
      ring_pop_front(r);
      any = true;
      continue;
    }
    RingEvent* d = r.segs.front().done;
    if (!d) break;  // a plan still being built (possibly the caller): cannot wait for it
    cudaError_t e = wait ? cudaEventSynchronize(d->ev) : cudaEventQuery(d->ev);
    if (e != cudaSuccess) {
      if (e != cudaErrorNotReady) cudaGetLastError();
      break;
    }
    ring_pop_front(r);
    any = true;
    wait = false;
  }
  if (r.segs.empty()) r.head = 0;
  return any;
}
char* ring_alloc(PinnedRing& r, size_t n, const tn_plan* owner) {
  n = (n + 255) & ~size_t(255);
  if (n > STAGE_MAX) return nullptr;
  if (!r.base) {
    if (r.tried) return nullptr;
    r.tried = true;
    if (cudaHostAlloc(reinterpret_cast<void**>(&r.base), RING_BYTES, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      r.base = nullptr;
      return nullptr;
    }
  }
  for (int attempt = 0; attempt < 64; ++attempt) {
    size_t at = SIZE_MAX;
    if (r.segs.empty()) {
      at = 0;
    } else {
      const size_t tail = r.segs.front().start;
      if (r.head >= tail) {                       // live data in [tail, head)
        if (r.head + n <= RING_BYTES) at = r.head;
        else if (n <= tail) at = 0;              // wrap
      } else if (r.head + n <= tail) {            // wrapped: live data in [tail, end) and [0, head)
        at = r.head;
      }
    }
    if (at != SIZE_MAX) {
      r.segs.push_back(RingSeg{at, at + n, owner, nullptr, false});
      r.head = at + n;
      return r.base + at;
    }
    // full: first take back whatever has completed, then wait for the oldest sealed range
    if (!ring_reclaim(r, false) && !ring_reclaim(r, true)) return nullptr;   // oldest unsealed: go pageable
  }
  return nullptr;
}
}  // namespace

cudaError_t plan_h2d(tn_plan* p, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  const void* from = src;
  static const bool pageable = getenv("TN_PAGEABLE_UPLOADS") != nullptr;   // A/B: the driver's own staging
  if (!pageable) {
    PinnedRing& r = ring();
    std::lock_guard<std::mutex> lk(r.mu);
    if (char* slot = ring_alloc(r, bytes, p)) {
      std::memcpy(slot, src, bytes);
      from = slot;
      ++p->n_staged;
    }
  }
  return cudaMemcpyAsync(dst, from, bytes, cudaMemcpyHostToDevice, p->plan_stream);
}

cudaError_t plan_h2d_parts(tn_plan* p, char* dst_base, const H2DPart* parts, int n, size_t total) {
  static const bool pageable = getenv("TN_PAGEABLE_UPLOADS") != nullptr;
  if (!pageable && total > 0) {
    char* slot = nullptr;
    {
      PinnedRing& r = ring();
      std::lock_guard<std::mutex> lk(r.mu);
      slot = ring_alloc(r, total, p);
      if (slot) {
        for (int i = 0; i < n; ++i) std::memcpy(slot + parts[i].off, parts[i].src, parts[i].bytes);
        ++p->n_staged;
      }
    }
    if (slot) return cudaMemcpyAsync(dst_base, slot, total, cudaMemcpyHostToDevice, p->plan_stream);
  }
  for (int i = 0; i < n; ++i) {
    if (!parts[i].bytes) continue;
    const cudaError_t e = cudaMemcpyAsync(dst_base + parts[i].off, parts[i].src, parts[i].bytes,
                                          cudaMemcpyHostToDevice, p->plan_stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void plan_h2d_seal(tn_plan* p) {
  if (p->n_staged == 0) return;
  PinnedRing& r = ring();
  std::lock_guard<std::mutex> lk(r.mu);
  RingEvent* d = nullptr;
  if (!r.free_ev.empty()) {
    d = r.free_ev.back();
    r.free_ev.pop_back();
  } else {
    d = new (std::nothrow) RingEvent();
    if (d && cudaEventCreateWithFlags(&d->ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      delete d;
      d = nullptr;
    }
  }
  if (d && cudaEventRecord(d->ev, p->plan_stream) != cudaSuccess) {
    cudaGetLastError();
    r.free_ev.push_back(d);
    d = nullptr;
  }
  if (!d) {  // cannot fence the staged uploads: wait for them on the host, then the ranges are free at once
    cudaStreamSynchronize(p->plan_stream);
    cudaGetLastError();
  }
  for (RingSeg& g : r.segs)
    if (g.owner == p && !g.done && !g.complete) {
      if (d) {
        g.done = d;
        ++d->refs;
      } else {
        g.complete = true;
      }
    }
  if (d && d->refs == 0) r.free_ev.push_back(d);
  p->n_staged = 0;
}

void shell_release(const PlanShell& sh) {
  if (!sh.stream) return;
  std::lock_guard<std::mutex> lk(g_shell_mu);
  g_shells.push_back(sh);
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
