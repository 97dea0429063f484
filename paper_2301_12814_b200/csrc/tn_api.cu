// C-ABI glue of libtn_theta.so: plan construction (K1 + host work decomposition), queries, the U
// builder entry point, exec (K3 → K4 → K5) and the row-sharded exec over NCCL. See
// include/tn_theta.h for the contract of every entry point and DESIGN.md for the design.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>

#include <cstdlib>
#include <chrono>

#include <dlfcn.h>

#include "tn_internal.cuh"

namespace tn {

static thread_local std::string g_last_error;

void set_error(const std::string& s) { g_last_error = s; }

tn_status fail(tn_status st, const std::string& s) {
  g_last_error = s;
  return st;
}

tn_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TN_OK;
  // the failure is reported through the returned status: take it out of the runtime's per-thread last-error
  // slot, or the next launch check of ANY later call would report it again as its own (a sticky error keeps
  // failing every later call regardless)
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) return fail(TN_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  return fail(TN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------------------------
// Work model shared by the shard split and the flop counters.
// ---------------------------------------------------------------------------------------------
struct Counts {
  int d, N;
  std::vector<int64_t> nl, nc, nr;
};

// Per-row work of a left row of charge q (prefix sums, O((N+1)·d) for all q):
//   fc[q] = 8 Σ_{c_c ∈ [q−d+1, q], n_c > 0} n_c(c_c) · cols(c_c)        (its K4 contraction flops, 8 per CMAC)
//   fm[q] = 8 Σ_{c_r} n_r(c_r) · #c · #non-empty c_c                     (its U-mix flops)
//   el[q] = Σ_{c ∈ [q−d+1, q]} C_c                                        (its Θ elements: K5 moves 32 B each)
struct RowCosts {
  std::vector<double> fc, fm, el;
};
static void row_costs(const Counts& k, RowCosts& rc) {
  const int d = k.d, N = k.N;
  std::vector<int64_t> pr(N + 2, 0), pc(N + 2, 0), pz(N + 2, 0);
  for (int q = 0; q <= N; ++q) {
    pr[q + 1] = pr[q] + k.nr[q];
    pc[q + 1] = pc[q] + k.nc[q];
    pz[q + 1] = pz[q] + (k.nc[q] > 0);
  }
  auto cols = [&](int c) { return (double)(pr[c + 1] - pr[std::max(0, c - d + 1)]); };  // C_c
  rc.fc.assign(N + 1, 0.0);
  rc.fm.assign(N + 1, 0.0);
  rc.el.assign(N + 1, 0.0);
  for (int q = 0; q <= N; ++q) {
    for (int cc = std::max(0, q - d + 1); cc <= q; ++cc) {
      rc.el[q] += cols(cc);
      if (k.nc[cc]) rc.fc[q] += 8.0 * (double)k.nc[cc] * cols(cc);
    }
    for (int cr = std::max(0, q - 2 * d + 2); cr <= q; ++cr) {
      const int lo = std::max(cr, q - d + 1), hi = std::min(q, cr + d - 1);
      if (hi < lo || !k.nr[cr]) continue;
      rc.fm[q] += 8.0 * (double)k.nr[cr] * (double)(hi - lo + 1) * (double)(pz[hi + 1] - pz[lo]);
    }
  }
}

// Shard bounds balance the estimated DEVICE TIME per row rather than raw flops: K4 turns
// contraction flops into time at ~41 TFLOP/s (useful, 3M form), K5 moves 32 B per Θ element at ~3.7 TB/s, so a
// Θ element weighs KAPPA ≈ 32·41/3.7 ≈ 355 flop-equivalents; the mix flops themselves ride on the memory-bound K5.
constexpr double KAPPA_EL = 355.0;
static void shard_bounds(const Counts& k, const RowCosts& rc, int world, std::vector<int64_t>& bounds) {
  std::vector<double> cost(k.N + 1);
  double total = 0.0;
  int64_t chi_l = 0;
  for (int q = 0; q <= k.N; ++q) {
    cost[q] = rc.fc[q] + KAPPA_EL * rc.el[q];
    total += cost[q] * (double)k.nl[q];
    chi_l += k.nl[q];
  }
  bounds.assign(world + 1, 0);
  bounds[world] = chi_l;
  // bounds[r] = first sorted row whose prefix cost (over the rows before it) reaches r/world of the total; the rows
  // of one charge q all cost cost[q], so each boundary inside a segment is found in O(1)
  double prefix = 0.0;
  int64_t row = 0;
  int r = 1;
  for (int q = 0; q <= k.N && r < world; ++q) {
    const int64_t n = k.nl[q];
    if (!n) continue;
    while (r < world) {
      const double target = total * (double)r / world;
      int64_t i;
      if (prefix >= target) {
        i = 0;
      } else if (cost[q] > 0.0) {
        i = (int64_t)std::ceil((target - prefix) / cost[q]);
        while (i > 0 && prefix + (double)(i - 1) * cost[q] >= target) --i;   // guard the rounding of ceil
        while (i < n && prefix + (double)i * cost[q] < target) ++i;
      } else {
        i = n;
      }
      if (i >= n) break;               // reached in a later segment
      bounds[r++] = row + i;
    }
    prefix += cost[q] * (double)n;
    row += n;
  }
  while (r < world) bounds[r++] = row;
}

// Sector owners for TN_GATHER_SECTOR_OWNER: longest-processing-time assignment by
// element count R_c·C_c (largest first onto the least-loaded rank, ties to the lower rank/sector).
void sector_owners(const std::vector<int64_t>& sizes, int world, std::vector<int32_t>& owner) {
  const int n = (int)sizes.size();
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sizes[a] > sizes[b]; });
  std::vector<int64_t> load(world, 0);
  owner.assign(n, 0);
  for (int c : order) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    owner[c] = best;
    load[best] += sizes[c];
  }
}

static void free_plan(tn_plan* p) {
  if (!p) return;
  // a captured exec may be replayed on any stream: wait for every replay before the blocks are reused
  if (p->captured) cudaDeviceSynchronize();
  // the blocks become reusable once the last library work that touched them is done (ev_fence, recorded after
  // the plan's own uploads and after every later exec / U build / SVD); the pool takes the event over
  Fence* f = fence_adopt(p->ev_fence);
  p->ev_fence = nullptr;
  for (void* blk : {p->blk_oz, p->blk_lit, p->blk_p, p->blk_slab, p->blk_pack, p->blk_work, p->blk_tab})
    pool_release_fenced(blk, f);
  fence_release(f);
  PlanShell sh;
  sh.dev = p->dev;
  sh.stream = p->plan_stream;
  for (int i = 0; i < 8; ++i) sh.ev[i] = p->ev[i];
  sh.ev_ready = p->ev_ready;
  plan_h2d_seal(p);   // a plan that failed mid-build may still hold unsealed ranges of the upload ring
  shell_release(sh);   // stream + timing events go back to the shell pool
  delete p;
}

// Carves 256-byte aligned sub-buffers out of one pool block.
struct Carver {
  size_t off = 0;
  template <class T>
  size_t take(int64_t n) {
    const size_t at = off;
    off += ((size_t)n * sizeof(T) + 255) / 256 * 256;
    return at;
  }
};

static int sm_count_of(int dev) {
  static int cached[64] = {};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    n = 148;
  }
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

static bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

__global__ void k_set_sectors(const SectorPtrs ptrs, SecEntry* __restrict__ tab) {
  for (int c = threadIdx.x; c < ptrs.n; c += blockDim.x) {
    tab[c].out = ptrs.out[c];
    tab[c].src = ptrs.src[c];
  }
}

tn_status make_sector_params(const tn_plan* p, double* const* out, const double* const* src, int which, cudaStream_t s,
                             SectorParams* sp) {
  SectorPtrs ptrs;
  ptrs.n = p->nsec;
  for (int c = 0; c < p->nsec; ++c) {
    ptrs.out[c] = reinterpret_cast<double2*>(out[c]);
    ptrs.src[c] = src ? reinterpret_cast<const double2*>(src[c]) : nullptr;
  }
  k_set_sectors<<<1, 256, 0, s>>>(ptrs, p->d_sec[which]);
  tn_status st = cuda_check(cudaGetLastError(), "sector table");
  sp->sec = p->d_sec[which];
  sp->ustart = p->d_ustart;
  sp->d = p->d;
  sp->N = p->N;
  return st;
}

// static part of the sector tables + the packed-U offsets, uploaded once per plan (both tables)
static tn_status upload_sector_tables(tn_plan* p) {
  p->h_sec.assign(p->nsec, SecEntry{});
  for (int c = 0; c < p->nsec; ++c) {
    SecEntry& e = p->h_sec[c];
    e.lrow0 = p->lrow0[c];
    e.col0 = p->col0[c];
    e.ld = (int32_t)p->C[c];
    // the mix reads P_{c_c} iff seg_c(c_c) is non-empty: exactly then K4 ran group c_c for every local row that
    // can need it (a row of Θ(c_c) in this shard); pair plans: one entry per centre KEY
    e.nonempty = p->off[1][c + 1] > p->off[1][c];
  }
  for (int w = 0; w < 2; ++w) {
    tn_status st = cuda_check(plan_h2d(p, p->d_sec[w], p->h_sec.data(), p->nsec * sizeof(SecEntry)), "H2D sector table");
    if (st != TN_OK) return st;
  }
  return cuda_check(plan_h2d(p, p->d_ustart, p->ustart.data(), p->ustart.size() * sizeof(int32_t)), "H2D U offsets");
}

}  // namespace tn

using namespace tn;

extern "C" {

const char* tn_status_string(tn_status s) {
  switch (s) {
    case TN_OK: return "TN_OK";
    case TN_ERR_DOMAIN: return "TN_ERR_DOMAIN";
    case TN_ERR_DIMENSION: return "TN_ERR_DIMENSION";
    case TN_ERR_CONSISTENCY: return "TN_ERR_CONSISTENCY";
    case TN_ERR_CUDA: return "TN_ERR_CUDA";
    case TN_ERR_OOM: return "TN_ERR_OOM";
    case TN_ERR_NCCL: return "TN_ERR_NCCL";
    case TN_ERR_UNSUPPORTED: return "TN_ERR_UNSUPPORTED";
  }
  return "TN_ERR_UNKNOWN";
}

const char* tn_last_error(void) { return g_last_error.c_str(); }

int tn_version(void) { return (0 << 16) | 1; }

tn_status tn_shard_rows_host(int d, int N, const int64_t* n_l, const int64_t* n_c, const int64_t* n_r,
                             int world_size, int64_t* bounds) {
  if (d < 2 || N < 0 || N > TN_MAX_N || world_size < 1) return fail(TN_ERR_DOMAIN, "tn_shard_rows_host: bad d/N/world");
  if (!n_l || !n_c || !n_r || !bounds) return fail(TN_ERR_DIMENSION, "tn_shard_rows_host: NULL pointer");
  Counts k{d, N, std::vector<int64_t>(n_l, n_l + N + 1), std::vector<int64_t>(n_c, n_c + N + 1),
           std::vector<int64_t>(n_r, n_r + N + 1)};
  for (int q = 0; q <= N; ++q)
    if (k.nl[q] < 0 || k.nc[q] < 0 || k.nr[q] < 0) return fail(TN_ERR_DOMAIN, "tn_shard_rows_host: negative count");
  std::vector<int64_t> b;
  RowCosts rc;
  row_costs(k, rc);
  shard_bounds(k, rc, world_size, b);
  std::copy(b.begin(), b.end(), bounds);
  return TN_OK;
}

tn_status tn_sector_owners_host(int n_sectors, const int64_t* sizes, int world_size, int32_t* owners) {
  if (n_sectors < 0 || world_size < 1) return fail(TN_ERR_DOMAIN, "tn_sector_owners_host: bad n/world");
  if ((n_sectors && (!sizes || !owners))) return fail(TN_ERR_DIMENSION, "tn_sector_owners_host: NULL");
  std::vector<int64_t> sz(sizes, sizes + n_sectors);
  std::vector<int32_t> o;
  sector_owners(sz, world_size, o);
  std::copy(o.begin(), o.end(), owners);
  return TN_OK;
}

tn_status tn_plan_sector_owner(const tn_plan* p, int c, int* owner) {
  if (!p || !owner) return fail(TN_ERR_DIMENSION, "tn_plan_sector_owner: NULL");
  if (c < 0 || c >= p->nsec) return fail(TN_ERR_DOMAIN, "tn_plan_sector_owner: sector out of range");
  *owner = p->owner.empty() ? 0 : p->owner[c];
  return TN_OK;
}

// packed U layout (SURVEY.md §8(c) "Packed U")
static void u_layout(tn_plan* p) {
  const int nmax = std::min(p->N, 2 * p->d - 2);
  int64_t tot = 0;
  p->ustart.clear();
  for (int n = 0; n <= nmax; ++n) {
    const int s = std::min(n, p->d - 1) - std::max(0, n - p->d + 1) + 1;
    p->ustart.push_back((int32_t)tot);
    tot += (int64_t)s * s;
  }
  p->u_size = tot;
}

// TN_PLAN_PROFILE=1: host µs per phase of tn_theta_plan on stderr (tools/plan_profile.py)
static bool plan_prof() {
  static const bool on = getenv("TN_PLAN_PROFILE") != nullptr;
  return on;
}
static double plan_now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define TN_PT(i) \
  if (plan_prof()) pt[i] = plan_now_us()

static tn_status plan_impl(int d, int N, int64_t chi_l, int64_t chi_c, int64_t chi_r, const int32_t* q_l,
                           const int32_t* q_c, const int32_t* q_r, const int32_t* const* q2, int world_size, int rank,
                           tn_plan** out) {
  if (!out) return fail(TN_ERR_DIMENSION, "tn_theta_plan: out is NULL");
  *out = nullptr;
  if (d < 2) return fail(TN_ERR_DOMAIN, "tn_theta_plan: d < 2");
  if (N < 0 || N > TN_MAX_N) return fail(TN_ERR_DOMAIN, "tn_theta_plan: N outside [0, TN_MAX_N]");
  if (chi_l < 1 || chi_c < 1 || chi_r < 1) return fail(TN_ERR_DOMAIN, "tn_theta_plan: bond dimension < 1");
  if (chi_l > INT32_MAX || chi_c > INT32_MAX || chi_r > INT32_MAX)
    return fail(TN_ERR_UNSUPPORTED, "tn_theta_plan: bond dimension > INT32_MAX");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(TN_ERR_DOMAIN, "tn_theta_plan: bad world_size/rank");
  if (!q_l || !q_c || !q_r) return fail(TN_ERR_DIMENSION, "tn_theta_plan: NULL charge array");
  if (std::min(N + 1, d) > TN_MAX_MIX) return fail(TN_ERR_UNSUPPORTED, "tn_theta_plan: min(N+1, d) > TN_MAX_MIX");
  if (q2) {
    if (!q2[0] || !q2[1] || !q2[2]) return fail(TN_ERR_DIMENSION, "tn_theta2_plan: NULL charge array");
    if ((N + 1) * (N + 1) > MAX_SEC)
      return fail(TN_ERR_UNSUPPORTED, "tn_theta2_plan: (N+1)^2 charge pairs exceed this build's sector limit (N <= 31)");
  }

  tn_plan* p = new (std::nothrow) tn_plan();
  if (!p) return fail(TN_ERR_OOM, "tn_theta_plan: host allocation");
  double pt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  TN_PT(0);
  p->d = d;
  p->N = N;
  p->world = world_size;
  p->rank = rank;
  p->chi[0] = chi_l;
  p->chi[1] = chi_c;
  p->chi[2] = chi_r;
  p->max_mix = std::min(N + 1, d);
  p->pair = q2 != nullptr;
  p->nq = p->pair ? (N + 1) * (N + 1) : N + 1;
  p->nsec = p->nq;
  tn_status st = TN_OK;
  int dev = 0;
  int32_t* d_q[3] = {nullptr, nullptr, nullptr};
  const int32_t* qs_in[3] = {q_l, q_c, q_r};
  cudaError_t aerr = cudaSuccess;
  Carver ct;
  size_t o_perm[3], o_qs[3], o_off[3], o_err, o_q[3] = {0, 0, 0}, o_q2[3] = {0, 0, 0};
  bool host_q[3], host_q2[3] = {false, false, false};
  bool all_host = true;
  int32_t* d_err = nullptr;
  const int nmax_u = std::min(N, 2 * d - 2);
  size_t o_bin = 0, o_sec[2] = {0, 0}, o_ust = 0;
  size_t up_bytes = 0;   // the leading, host-provided part of the table block (one upload)
  std::vector<double2> hbin((size_t)(nmax_u + 1) * (nmax_u + 1), double2{0.0, 0.0});
#define TN_TRY(expr, what)                      \
  do {                                          \
    st = cuda_check((expr), what);              \
    if (st != TN_OK) goto done;                 \
  } while (0)
  // a non-sticky error left in this thread's last-error slot by an earlier, already reported failure must not be
  // reported again by the launch checks below as if this plan's K1 had failed; a sticky one fails them anyway
  cudaGetLastError();
  TN_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  p->dev = dev;
  p->sm_count = sm_count_of(dev);
  {
    PlanShell sh;
    TN_TRY(shell_acquire(&sh), "plan stream");
    p->plan_stream = sh.stream;
    for (int i = 0; i < 8; ++i) p->ev[i] = sh.ev[i];
    p->ev_ready = sh.ev_ready;
  }
  TN_TRY(cudaEventCreateWithFlags(&p->ev_fence, cudaEventDisableTiming), "event create");
  TN_PT(1);
  // ---- one pool block for the bond tables (+ staging of host charges) ----
  // layout: the host-provided part first — error flags (uploaded as zeros), binomials, host charges — so it goes
  // up as ONE staged copy; then the device-built tables
  for (int b = 0; b < 3; ++b) {
    host_q[b] = !is_device_ptr(qs_in[b]);
    all_host = all_host && host_q[b];
    if (q2) {
      host_q2[b] = !is_device_ptr(q2[b]);
      all_host = all_host && host_q2[b];
    }
  }
  o_err = ct.take<int32_t>(4);
  o_bin = ct.take<double2>((int64_t)(nmax_u + 1) * (nmax_u + 1));
  for (int b = 0; b < 3; ++b) {
    if (host_q[b]) o_q[b] = ct.take<int32_t>(p->chi[b]);
    if (q2 && host_q2[b]) o_q2[b] = ct.take<int32_t>(p->chi[b]);
  }
  up_bytes = ct.off;
  for (int b = 0; b < 3; ++b) {
    o_perm[b] = ct.take<int32_t>(p->chi[b]);
    o_qs[b] = ct.take<int32_t>(p->chi[b]);
    o_off[b] = ct.take<int32_t>(p->nq + 1);
  }
  o_sec[0] = ct.take<SecEntry>(p->nq);
  o_sec[1] = ct.take<SecEntry>(p->nq);
  o_ust = ct.take<int32_t>(nmax_u + 1);
  for (int n = 0; n <= nmax_u; ++n) {  // exact C(n,k) as a double-double pair (n ≤ TN_MAX_N)
    unsigned __int128 c = 1;
    for (int k = 0; k <= n; ++k) {
      if (k > 0) c = c * (unsigned __int128)(n - k + 1) / (unsigned __int128)k;
      const double hi = (double)c;
      const unsigned __int128 hi_i = (unsigned __int128)hi;
      const double lo = c >= hi_i ? (double)(c - hi_i) : -(double)(hi_i - c);
      hbin[(size_t)n * (nmax_u + 1) + k] = double2{hi, lo};
    }
  }
  TN_PT(2);
  p->blk_tab = pool_alloc(ct.off, &aerr);
  TN_PT(3);
  TN_TRY(aerr, "pool alloc (bond tables)");
  {
    char* base = static_cast<char*>(p->blk_tab);
    SortArgs sa{};
    for (int b = 0; b < 3; ++b) {
      p->d_perm[b] = reinterpret_cast<int32_t*>(base + o_perm[b]);
      p->d_qs[b] = reinterpret_cast<int32_t*>(base + o_qs[b]);
      p->d_off[b] = reinterpret_cast<int32_t*>(base + o_off[b]);
      const int32_t* src = qs_in[b];
      if (host_q[b]) {
        d_q[b] = reinterpret_cast<int32_t*>(base + o_q[b]);
        src = d_q[b];
      }
      sa.q[b] = src;
      sa.q2[b] = q2 ? q2[b] : nullptr;
      if (q2 && host_q2[b]) sa.q2[b] = reinterpret_cast<int32_t*>(base + o_q2[b]);
      sa.chi[b] = p->chi[b];
      sa.perm[b] = p->d_perm[b];
      sa.qs[b] = p->d_qs[b];
      sa.off[b] = p->d_off[b];
    }
    d_err = reinterpret_cast<int32_t*>(base + o_err);
    p->d_rowperm = p->d_perm[0];  // single-charge groups index sorted positions directly
    p->n_rowlist = p->chi[0];
    p->d_colperm = p->d_perm[2];
    sa.err = d_err;
    p->d_binom = reinterpret_cast<double2*>(base + o_bin);
    p->d_sec[0] = reinterpret_cast<SecEntry*>(base + o_sec[0]);
    p->d_sec[1] = reinterpret_cast<SecEntry*>(base + o_sec[1]);
    p->d_ustart = reinterpret_cast<int32_t*>(base + o_ust);
    {  // error flags (zero), binomials and host charges: one staged upload of the block's leading region
      static const int32_t zeros[4] = {0, 0, 0, 0};
      std::vector<H2DPart> parts;
      parts.push_back(H2DPart{o_err, zeros, sizeof(zeros)});
      parts.push_back(H2DPart{o_bin, hbin.data(), hbin.size() * sizeof(double2)});
      for (int b = 0; b < 3; ++b) {
        if (host_q[b]) parts.push_back(H2DPart{o_q[b], qs_in[b], (size_t)p->chi[b] * sizeof(int32_t)});
        if (q2 && host_q2[b]) parts.push_back(H2DPart{o_q2[b], q2[b], (size_t)p->chi[b] * sizeof(int32_t)});
      }
      TN_TRY(plan_h2d_parts(p, base, parts.data(), (int)parts.size(), up_bytes), "H2D charges / binomials");
    }
    // ---- K1: sort each bond by charge (one launch, one CTA per bond) ----
    TN_TRY(cudaEventRecord(p->ev[0], p->plan_stream), "event");
    TN_TRY(launch_sort_bonds(sa, N, p->plan_stream), "K1 launch");
    TN_PT(4);
    TN_TRY(cudaEventRecord(p->ev[1], p->plan_stream), "event");
    p->rec_k1 = true;
  }
  if (all_host) {
    // host charges: the offset tables are counted here (the same stable counting-sort definition K1 applies
    // on the device for perm), so the plan never waits for the GPU — the tables below go up asynchronously
    // and the next gate's planning overlaps this gate's kernels
    for (int b = 0; b < 3; ++b) {
      std::vector<int32_t>& o = p->off[b];
      o.assign(p->nq + 1, 0);
      const int32_t* a = qs_in[b];
      const int32_t* a2 = q2 ? q2[b] : nullptr;
      bool bad = false;
      int32_t* hist = o.data() + 1;
      if (!a2) {
        // four interleaved histograms: charge-sorted input hits one bin many times in a row, and a single
        // histogram serialises those increments on store-to-load forwarding
        std::vector<int32_t> h4(4 * (size_t)p->nq, 0);
        const int64_t n = p->chi[b];
        int64_t i = 0;
        for (; i + 4 <= n; i += 4) {
          uint32_t x[4];
          for (int u = 0; u < 4; ++u) {
            x[u] = (uint32_t)a[i + u];
            bad |= x[u] > (uint32_t)N;
          }
          for (int u = 0; u < 4; ++u) h4[u * (size_t)p->nq + (x[u] > (uint32_t)N ? 0 : x[u])]++;
        }
        for (; i < n; ++i) {
          const uint32_t x = (uint32_t)a[i];
          bad |= x > (uint32_t)N;
          h4[x > (uint32_t)N ? 0 : x]++;
        }
        for (int k = 0; k < p->nq; ++k) hist[k] = h4[k] + h4[p->nq + k] + h4[2 * p->nq + k] + h4[3 * p->nq + k];
      } else {
        for (int64_t i = 0; i < p->chi[b]; ++i) {
          const uint32_t x = (uint32_t)a[i], y = (uint32_t)a2[i];
          const bool oob = x > (uint32_t)N || y > (uint32_t)N;
          bad |= oob;
          hist[oob ? 0 : x * (N + 1) + y]++;
        }
      }
      if (bad) {
        st = fail(TN_ERR_DOMAIN, "tn_theta_plan: a bond charge lies outside [0, N]");
        goto done;
      }
      for (int k = 0; k < p->nq; ++k) o[k + 1] += o[k];
    }
  } else {
    // device charges: one D2H of off[3] + err after K1 (the call's only host synchronisation)
    int32_t herr[4] = {0, 0, 0, 0};
    for (int b = 0; b < 3; ++b) p->off[b].resize(p->nq + 1);
    for (int b = 0; b < 3; ++b)
      TN_TRY(cudaMemcpyAsync(p->off[b].data(), p->d_off[b], (p->nq + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             p->plan_stream), "D2H off");
    TN_TRY(cudaMemcpyAsync(herr, d_err, sizeof(herr), cudaMemcpyDeviceToHost, p->plan_stream), "D2H err");
    TN_TRY(cudaStreamSynchronize(p->plan_stream), "K1 sync");
    if (herr[0] || herr[1] || herr[2]) {
      st = fail(TN_ERR_DOMAIN, "tn_theta_plan: a bond charge lies outside [0, N]");
      goto done;
    }
  }
  TN_PT(5);
  if (p->pair) {
    // ---- MPO pair plan: sectors, groups, two-pass mix (tn_pair.cu) ----
    st = build_pair_tables(p);
    if (st != TN_OK) goto done;
    {
      std::vector<int64_t> sizes(p->nsec);
      for (int c = 0; c < p->nsec; ++c) sizes[c] = p->R[c] * p->C[c];
      sector_owners(sizes, world_size, p->owner);
    }
    p->ws_bytes += (int64_t)ct.off;
    u_layout(p);
    if ((st = upload_sector_tables(p)) != TN_OK) goto done;
    plan_h2d_seal(p);
    TN_TRY(cudaEventRecord(p->ev_ready, p->plan_stream), "plan tables ready");
    TN_TRY(plan_touch(p, p->plan_stream), "plan fence");
  } else {
    // ---- sectors (R2) ----
    const auto& ol = p->off[0];
    const auto& oc = p->off[1];
    const auto& orr = p->off[2];
    Counts k{d, N, std::vector<int64_t>(N + 1), std::vector<int64_t>(N + 1), std::vector<int64_t>(N + 1)};
    for (int q = 0; q <= N; ++q) {
      k.nl[q] = ol[q + 1] - ol[q];
      k.nc[q] = oc[q + 1] - oc[q];
      k.nr[q] = orr[q + 1] - orr[q];
    }
    RowCosts rc;
    row_costs(k, rc);
    shard_bounds(k, rc, world_size, p->bounds);
    p->r0 = p->bounds[rank];
    p->r1 = p->bounds[rank + 1];
    {  // this rank's share of the useful work (rows [r0, r1))
      double lc = 0.0, lm = 0.0;
      for (int q = 0; q <= N; ++q) {
        const int64_t a = std::max<int64_t>(ol[q], p->r0), b = std::min<int64_t>(ol[q + 1], p->r1);
        if (b <= a) continue;
        lc += rc.fc[q] * (double)(b - a);
        lm += rc.fm[q] * (double)(b - a);
      }
      p->f_contract_local = (int64_t)llround(lc);
      p->f_mix_local = (int64_t)llround(lm);
    }
    p->R.resize(N + 1);
    p->C.resize(N + 1);
    p->row0.resize(N + 1);
    p->col0.resize(N + 1);
    p->lR.resize(N + 1);
    p->lrow0.resize(N + 1);
    for (int c = 0; c <= N; ++c) {
      const int64_t a0 = ol[c], a1 = ol[std::min(N, c + d - 1) + 1];
      const int64_t b0 = orr[std::max(0, c - d + 1)], b1 = orr[c + 1];
      p->row0[c] = a0;
      p->R[c] = a1 - a0;
      p->col0[c] = b0;
      p->C[c] = b1 - b0;
      const int64_t l0 = std::min(std::max(a0, p->r0), p->r1), l1 = std::min(std::max(a1, p->r0), p->r1);
      p->lrow0[c] = l0;
      p->lR[c] = l1 - l0;
      if (p->C[c] > INT32_MAX || p->R[c] > INT32_MAX) {
        st = fail(TN_ERR_UNSUPPORTED, "sector dimension > INT32_MAX");
        goto done;
      }
    }
    {
      std::vector<int64_t> sizes(N + 1);
      for (int c = 0; c <= N; ++c) sizes[c] = p->R[c] * p->C[c];
      sector_owners(sizes, world_size, p->owner);
    }
    // ---- useful flops of the whole problem ----
    // for a (c_l, c_r) block the valid c (= c_c) form the range [max(c_r, c_l−d+1), min(c_l, c_r+d−1)]: prefix
    // sums over n_c and over [n_c > 0] give Σ n_c and #non-empty c_c in O(1) per block
    {
      std::vector<int64_t> pc(N + 2, 0), pz(N + 2, 0);
      for (int q = 0; q <= N; ++q) {
        pc[q + 1] = pc[q] + k.nc[q];
        pz[q + 1] = pz[q] + (k.nc[q] > 0);
      }
      for (int cl = 0; cl <= N; ++cl) {
        if (!k.nl[cl]) continue;
        for (int cr = std::max(0, cl - 2 * d + 2); cr <= cl; ++cr) {
          const int lo = std::max(cr, cl - d + 1), hi = std::min(cl, cr + d - 1);
          if (hi < lo || !k.nr[cr]) continue;
          const int64_t nvc = hi - lo + 1, nvcc = pz[hi + 1] - pz[lo];
          p->f_contract += 8 * k.nl[cl] * k.nr[cr] * (pc[hi + 1] - pc[lo]);
          p->f_mix += 8 * k.nl[cl] * k.nr[cr] * nvc * nvcc;
        }
      }
    }
    // ---- groups: one per center charge with a non-empty segment and local rows ----
    int64_t a_off = 0, b_off = 0;
    for (int cc = 0; cc <= N; ++cc) {
      const int64_t K = oc[cc + 1] - oc[cc];
      if (K == 0 || p->lR[cc] == 0 || p->C[cc] == 0) continue;
      GroupDesc g{};
      g.cc = cc;
      g.row0 = p->lrow0[cc];
      g.col0 = p->col0[cc];
      g.k0 = oc[cc];
      g.R = (int32_t)p->lR[cc];
      g.C = (int32_t)p->C[cc];
      g.K = (int32_t)K;
      g.K4 = (int32_t)((K + 3) / 4 * 4);
      g.nmt = (g.R + BM - 1) / BM;
      g.nnt = (g.C + BN - 1) / BN;
      g.a_off = a_off;
      g.b_off = b_off;
      a_off += (int64_t)g.nmt * BM * g.K4;
      b_off += (int64_t)g.nnt * BN * g.K4;
      p->f_exec += 8 * (int64_t)g.nmt * BM * (int64_t)g.nnt * BN * g.K4;
      p->groups.push_back(g);
    }
    p->a_elems = a_off;
    p->b_elems = b_off;
    TN_PT(6);
    // ---- tile list, heavy-first (longest K first) ----
    std::vector<int> order(p->groups.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p->groups[x].K4 > p->groups[y].K4; });
    std::vector<TileDesc>& tiles = p->h_tiles;
    {
      int64_t nt_all = 0;
      for (const auto& g : p->groups) nt_all += (int64_t)g.nmt * g.nnt;
      tiles.resize((size_t)nt_all);
      TileDesc* t = tiles.data();
      for (int gi : order) {
        const auto& g = p->groups[gi];
        for (int mt = 0; mt < g.nmt; ++mt)
          for (int nt = 0; nt < g.nnt; ++nt) *t++ = TileDesc{gi, mt, nt, 0};
      }
    }
    p->ntiles = (int64_t)tiles.size();
    std::vector<MixTile>& mix = p->h_mix;
    build_mix_tiles(p, mix);
    TN_PT(7);
    p->nmix = (int64_t)mix.size();
    if (!p->groups.empty() || !mix.empty()) {
      Carver cw;
      const size_t o_g = cw.take<GroupDesc>((int64_t)p->groups.size());
      const size_t o_t = cw.take<TileDesc>((int64_t)tiles.size());
      const size_t o_m = cw.take<MixTile>((int64_t)mix.size());
      const size_t o_a = cw.take<double2>(p->a_elems);
      const size_t o_b = cw.take<double2>(p->b_elems);
      p->blk_work = pool_alloc(cw.off, &aerr);
      TN_PT(8);
      TN_TRY(aerr, "pool alloc (workspace)");
      char* base = static_cast<char*>(p->blk_work);
      p->d_groups = reinterpret_cast<GroupDesc*>(base + o_g);
      p->d_tiles = reinterpret_cast<TileDesc*>(base + o_t);
      p->d_mix = reinterpret_cast<MixTile*>(base + o_m);
      p->d_apanel = reinterpret_cast<double2*>(base + o_a);
      p->d_bpanel = reinterpret_cast<double2*>(base + o_b);
      if (!p->groups.empty()) {
        TN_TRY(plan_h2d(p, p->d_groups, p->groups.data(), p->groups.size() * sizeof(GroupDesc)), "H2D groups");
        TN_TRY(plan_h2d(p, p->d_tiles, tiles.data(), tiles.size() * sizeof(TileDesc)), "H2D tiles");
      }
      if (!mix.empty())
        TN_TRY(plan_h2d(p, p->d_mix, mix.data(), mix.size() * sizeof(MixTile)), "H2D mix tiles");
      // no host sync: tn_theta_exec's stream waits for ev_ready (the host vectors stay alive in the plan)
      p->ws_bytes = (int64_t)cw.off;
    }
    p->ws_bytes += (int64_t)ct.off;
    u_layout(p);
    if ((st = upload_sector_tables(p)) != TN_OK) goto done;
    plan_h2d_seal(p);
    TN_TRY(cudaEventRecord(p->ev_ready, p->plan_stream), "plan tables ready");
    TN_TRY(plan_touch(p, p->plan_stream), "plan fence");
    TN_PT(9);
    if (plan_prof())
      fprintf(stderr, "[plan] world %d rank %d us: shell %.1f sizing %.1f tab_alloc %.1f h2d+K1 %.1f count %.1f "
              "sectors+groups %.1f tiles+mix %.1f ws_alloc %.1f uploads %.1f total %.1f (tiles %lld mix %lld)\n",
              world_size, rank, pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[5] - pt[4],
              pt[6] - pt[5], pt[7] - pt[6], pt[8] - pt[7], pt[9] - pt[8], pt[9] - pt[0], (long long)p->ntiles,
              (long long)p->nmix);
  }
done:
#undef TN_TRY
  if (st != TN_OK) {
    free_plan(p);
    return st;
  }
  *out = p;
  return TN_OK;
}

tn_status tn_theta_plan(int d, int N, int64_t chi_l, int64_t chi_c, int64_t chi_r, const int32_t* q_l,
                        const int32_t* q_c, const int32_t* q_r, int world_size, int rank, tn_plan** out) {
  return plan_impl(d, N, chi_l, chi_c, chi_r, q_l, q_c, q_r, nullptr, world_size, rank, out);
}

tn_status tn_theta2_plan(int d, int N, int64_t chi_l, int64_t chi_c, int64_t chi_r, const int32_t* q1_l,
                         const int32_t* q2_l, const int32_t* q1_c, const int32_t* q2_c, const int32_t* q1_r,
                         const int32_t* q2_r, int world_size, int rank, tn_plan** out) {
  if (!q1_l || !q1_c || !q1_r) return fail(TN_ERR_DIMENSION, "tn_theta2_plan: NULL charge array");
  const int32_t* q2[3] = {q2_l, q2_c, q2_r};
  return plan_impl(d, N, chi_l, chi_c, chi_r, q1_l, q1_c, q1_r, q2, world_size, rank, out);
}

tn_status tn_plan_destroy(tn_plan* plan) {
  free_plan(plan);
  return TN_OK;
}

tn_status tn_plan_sector_shape(const tn_plan* p, int c, int64_t* R, int64_t* C) {
  if (!p || !R || !C) return fail(TN_ERR_DIMENSION, "tn_plan_sector_shape: NULL");
  if (c < 0 || c >= p->nsec) return fail(TN_ERR_DOMAIN, "tn_plan_sector_shape: sector outside [0, N] (pair plans: [0, (N+1)^2))");
  *R = p->R[c];
  *C = p->C[c];
  return TN_OK;
}

tn_status tn_plan_local_sector_shape(const tn_plan* p, int c, int64_t* R, int64_t* C, int64_t* row_begin) {
  if (!p || !R || !C || !row_begin) return fail(TN_ERR_DIMENSION, "tn_plan_local_sector_shape: NULL");
  if (c < 0 || c >= p->nsec) return fail(TN_ERR_DOMAIN, "tn_plan_local_sector_shape: sector out of range");
  *R = p->lR[c];
  *C = p->C[c];
  *row_begin = p->lrow0[c] - p->row0[c];
  return TN_OK;
}

tn_status tn_plan_perm(const tn_plan* p, int bond, int32_t* host_out) {
  if (!p || !host_out) return fail(TN_ERR_DIMENSION, "tn_plan_perm: NULL");
  if (bond < 0 || bond > 2) return fail(TN_ERR_DIMENSION, "tn_plan_perm: bond id");
  // K1 ran on the plan's own stream (and a host-charge plan never waited for it): copy on that stream
  tn_status st = cuda_check(cudaMemcpyAsync(host_out, p->d_perm[bond], p->chi[bond] * sizeof(int32_t),
                                            cudaMemcpyDeviceToHost, p->plan_stream), "tn_plan_perm D2H");
  if (st != TN_OK) return st;
  return cuda_check(cudaStreamSynchronize(p->plan_stream), "tn_plan_perm sync");
}

tn_status tn_plan_offsets(const tn_plan* p, int bond, int32_t* host_out) {
  if (!p || !host_out) return fail(TN_ERR_DIMENSION, "tn_plan_offsets: NULL");
  if (bond < 0 || bond > 2) return fail(TN_ERR_DIMENSION, "tn_plan_offsets: bond id");
  std::copy(p->off[bond].begin(), p->off[bond].end(), host_out);
  return TN_OK;
}

tn_status tn_plan_shard_rows(const tn_plan* p, int r, int64_t* r0, int64_t* r1) {
  if (!p || !r0 || !r1) return fail(TN_ERR_DIMENSION, "tn_plan_shard_rows: NULL");
  if (r < 0 || r >= p->world) return fail(TN_ERR_DOMAIN, "tn_plan_shard_rows: rank outside [0, world)");
  *r0 = p->bounds[r];
  *r1 = p->bounds[r + 1];
  return TN_OK;
}

tn_status tn_plan_flops(const tn_plan* p, int64_t* f_contract, int64_t* f_mix, int64_t* f_exec,
                        int64_t* f_contract_local, int64_t* f_mix_local) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_plan_flops: NULL");
  if (f_contract) *f_contract = p->f_contract;
  if (f_mix) *f_mix = p->f_mix;
  if (f_exec) *f_exec = p->contraction == TN_CONTRACT_PAPER_LITERAL ? p->lit_flops : p->f_exec;
  if (f_contract_local) *f_contract_local = p->f_contract_local;
  if (f_mix_local) *f_mix_local = p->f_mix_local;
  return TN_OK;
}

tn_status tn_plan_u_size(const tn_plan* p, int64_t* n) {
  if (!p || !n) return fail(TN_ERR_DIMENSION, "tn_plan_u_size: NULL");
  *n = p->u_size;
  return TN_OK;
}

tn_status tn_plan_workspace_bytes(const tn_plan* p, int64_t* bytes) {
  if (!p || !bytes) return fail(TN_ERR_DIMENSION, "tn_plan_workspace_bytes: NULL");
  *bytes = p->ws_bytes;
  return TN_OK;
}

tn_status tn_plan_set_contraction(tn_plan* p, int mode, int slices) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_plan_set_contraction: NULL plan");
  if (mode == TN_CONTRACT_F64_DMMA) {
    p->contraction = mode;
    return TN_OK;
  }
  if (mode == TN_CONTRACT_PAPER_LITERAL) {
    if (p->pair) return fail(TN_ERR_UNSUPPORTED, "tn_plan_set_contraction: the literal ablation is single-charge only");
    if (!p->blk_lit) {
      const tn_status st = build_literal(p);
      if (st != TN_OK) return st;
    }
    p->contraction = mode;
    return TN_OK;
  }
  if (mode != TN_CONTRACT_INT8_OZAKI) return fail(TN_ERR_DOMAIN, "tn_plan_set_contraction: unknown mode");
  if (slices < OZ_SMIN || slices > OZ_SMAX) return fail(TN_ERR_DOMAIN, "tn_plan_set_contraction: slices outside [4, 8]");
  if (p->blk_oz && p->oz_slices == slices) {
    p->contraction = mode;
    return TN_OK;
  }
  // exactness of the int32 diagonal accumulators (and of the S ≤ 6 int64 recombination) needs K ≤ 2048
  for (const auto& gd : p->groups)
    if (gd.K > OZ_KMAX)
      return fail(TN_ERR_UNSUPPORTED, "tn_plan_set_contraction: a centre charge segment exceeds 2048 bonds (INT8 emulation)");
  // (re)build the slice layout: same groups (center charges) as the DMMA path
  if (p->blk_oz) {
    // the previous layout's last use is fenced by ev_fence (the exec stream itself may no longer exist)
    if (cudaEventSynchronize(p->ev_fence) != cudaSuccess) cudaGetLastError();
    pool_release(p->blk_oz, nullptr, false);
    p->blk_oz = nullptr;
  }
  p->oz_groups.clear();
  int64_t a_off = 0, b_off = 0, ea = 0, eb = 0;
  p->oz_macs = 0;
  for (const auto& gd : p->groups) {
    OzGroup g{};
    g.cc = gd.cc;
    g.row0 = gd.row0;
    g.col0 = gd.col0;
    g.k0 = gd.k0;
    g.R = gd.R;
    g.C = gd.C;
    g.K = gd.K;
    g.Kp = (gd.K + OZ_BK - 1) / OZ_BK * OZ_BK;
    g.nmt = (g.R + OZ_BM - 1) / OZ_BM;
    g.nnt = (g.C + OZ_BN - 1) / OZ_BN;
    g.nkc = g.Kp / OZ_BK;
    g.a_off = a_off;
    g.b_off = b_off;
    g.ea_off = ea;
    g.eb_off = eb;
    a_off += (int64_t)g.nmt * g.nkc * 2 * slices * OZ_A_TILE;
    b_off += (int64_t)g.nnt * g.nkc * 3 * slices * OZ_B_TILE;
    ea += g.R;
    eb += g.C;
    p->oz_macs += (int64_t)g.nmt * g.nnt * 2 * g.nkc * (slices * (slices + 1) / 2) * 2 * OZ_BM * OZ_BN * OZ_BK;
    p->oz_groups.push_back(g);
  }
  std::vector<int> order(p->oz_groups.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p->oz_groups[x].Kp > p->oz_groups[y].Kp; });
  std::vector<OzTile>& tiles = p->h_oz_tiles;
  tiles.clear();
  for (int gi : order)
    for (int mt = 0; mt < p->oz_groups[gi].nmt; ++mt)
      for (int nt = 0; nt < p->oz_groups[gi].nnt; ++nt) tiles.push_back(OzTile{gi, mt, nt, 0});
  p->oz_ntiles = (int64_t)tiles.size();
  if (p->oz_groups.empty()) {
    p->oz_slices = slices;
    p->contraction = mode;
    return TN_OK;
  }
  Carver cw;
  const size_t o_g = cw.take<OzGroup>((int64_t)p->oz_groups.size());
  const size_t o_t = cw.take<OzTile>((int64_t)tiles.size());
  const size_t o_ea = cw.take<int32_t>(ea);
  const size_t o_eb = cw.take<int32_t>(eb);
  const size_t o_a = cw.take<int8_t>(a_off);
  const size_t o_b = cw.take<int8_t>(b_off);
  cudaError_t aerr = cudaSuccess;
  p->blk_oz = pool_alloc(cw.off, &aerr);
  if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (INT8 emulation workspace)");
  char* base = static_cast<char*>(p->blk_oz);
  p->d_oz_groups = reinterpret_cast<OzGroup*>(base + o_g);
  p->d_oz_tiles = reinterpret_cast<OzTile*>(base + o_t);
  p->d_oea = reinterpret_cast<int32_t*>(base + o_ea);
  p->d_oeb = reinterpret_cast<int32_t*>(base + o_eb);
  p->d_oa = reinterpret_cast<int8_t*>(base + o_a);
  p->d_ob = reinterpret_cast<int8_t*>(base + o_b);
  tn_status st = cuda_check(cudaMemcpyAsync(p->d_oz_groups, p->oz_groups.data(), p->oz_groups.size() * sizeof(OzGroup),
                                            cudaMemcpyHostToDevice, p->plan_stream), "H2D oz groups");
  if (st != TN_OK) return st;
  st = cuda_check(cudaMemcpyAsync(p->d_oz_tiles, tiles.data(), tiles.size() * sizeof(OzTile), cudaMemcpyHostToDevice,
                                  p->plan_stream), "H2D oz tiles");
  if (st != TN_OK) return st;
  st = cuda_check(cudaEventRecord(p->ev_ready, p->plan_stream), "oz tables ready");
  if (st == TN_OK) st = cuda_check(plan_touch(p, p->plan_stream), "plan fence");
  if (st != TN_OK) return st;
  p->ws_bytes += (int64_t)cw.off;
  p->oz_slices = slices;
  p->contraction = mode;
  return TN_OK;
}

tn_status tn_plan_get_contraction(const tn_plan* p, int* mode, int* slices) {
  if (!p || !mode || !slices) return fail(TN_ERR_DIMENSION, "tn_plan_get_contraction: NULL");
  *mode = p->contraction;
  *slices = p->contraction == TN_CONTRACT_INT8_OZAKI ? p->oz_slices : 0;
  return TN_OK;
}

tn_status tn_plan_reserve(const tn_plan* p, int32_t count) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_plan_reserve: NULL plan");
  for (const void* blk : {p->blk_tab, p->blk_work, p->blk_p, p->blk_slab, p->blk_pack, p->blk_oz, p->blk_lit}) {
    const cudaError_t e = pool_reserve_like(blk, count);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_check(e, "tn_plan_reserve");
    }
  }
  return TN_OK;
}

tn_status tn_plan_exec_launches(const tn_plan* p, int64_t* n_launches) {
  if (!p || !n_launches) return fail(TN_ERR_DIMENSION, "tn_plan_exec_launches: NULL");
  int64_t n = 0;
  if (p->contraction == TN_CONTRACT_PAPER_LITERAL) {
    n = p->lit_secs.empty() ? 0 : 2 + (p->lit_ntiles > 0);                 // K3L a/b, K4L
  } else {
    const bool emu = p->contraction == TN_CONTRACT_INT8_OZAKI;
    if (emu) n += (p->oz_groups.empty() ? 0 : 4) + (p->oz_ntiles > 0);      // K3O ×4, K4O
    else n += (p->groups.empty() ? 0 : 2) + (p->ntiles > 0);                  // K3 a/b, K4
    if (p->pair) {
      for (int ps = 0; ps < 2; ++ps)                                          // K5P, two passes × (single / multi-value tiles) × register class
        for (int m = 0; m < 2; ++m)
          for (int c = 0; c < 4; ++c) n += p->nmix2_grp[ps][m][c] > 0;                // one launch per class
      n += p->nmix_fused > 0;                                                          // K5F (short-vector blocks)
    } else {
      const int64_t c0 = p->nmix_cls[0], c1 = p->nmix_cls[1], c2 = p->nmix_cls[2], c3 = p->nmix - c0 - c1 - c2;
      n += (c0 > 0) + (c1 > 0) + (c2 > 0) + (c3 > 0);                        // K5, one launch per L class
    }
  }
  if (n > 0) ++n;   // k_set_sectors: the exec's output pointers into the plan's sector table
  *n_launches = n;
  return TN_OK;
}

tn_status tn_plan_kernel_times(const tn_plan* p, float* ms) {
  if (!p || !ms) return fail(TN_ERR_DIMENSION, "tn_plan_kernel_times: NULL");
  for (int i = 0; i < 5; ++i) ms[i] = -1.0f;
  auto span = [&](int a, int b, float* out) -> tn_status {
    tn_status st = cuda_check(cudaEventSynchronize(p->ev[b]), "event sync");
    if (st != TN_OK) return st;
    return cuda_check(cudaEventElapsedTime(out, p->ev[a], p->ev[b]), "event elapsed");
  };
  tn_status st = TN_OK;
  if (p->rec_k1 && (st = span(0, 1, &ms[0])) != TN_OK) return st;
  if (p->rec_k2 && (st = span(2, 3, &ms[1])) != TN_OK) return st;
  if (p->rec_exec) {
    if ((st = span(4, 5, &ms[2])) != TN_OK) return st;
    if ((st = span(5, 6, &ms[3])) != TN_OK) return st;
    if ((st = span(6, 7, &ms[4])) != TN_OK) return st;
  }
  return TN_OK;
}

// The exec stream waits for the plan's asynchronous table upload. Under CUDA graph capture that event lies
// outside the capture (waiting on it would invalidate the capture), and a replay may run on any stream, so
// the host waits for the upload instead and marks the plan captured: its blocks then go back to the pool
// only after a device-wide synchronisation (free_plan), because a replay's stream is unknown to the plan.
}  // extern "C"
namespace tn {
tn_status wait_tables(const tn_plan* p, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) cs = cudaStreamCaptureStatusNone;
  if (cs != cudaStreamCaptureStatusNone) {
    p->captured = true;
    // a host wait is a "potentially unsafe" call under global capture mode: relax this thread's mode for it
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    const cudaError_t e = cudaEventSynchronize(p->ev_ready);
    cudaThreadExchangeStreamCaptureMode(&mode);
    return cuda_check(e, "plan tables (captured exec)");
  }
  return cuda_check(cudaStreamWaitEvent(s, p->ev_ready, 0), "wait for plan tables");
}
}  // namespace tn
extern "C" {

tn_status tn_build_bs_unitary(const tn_plan* p, double theta, double phi, tn_stream stream, double* U_out) {
  if (!p || !U_out) return fail(TN_ERR_DIMENSION, "tn_build_bs_unitary: NULL");
  if (!std::isfinite(theta) || !std::isfinite(phi)) return fail(TN_ERR_DOMAIN, "tn_build_bs_unitary: non-finite angle");
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_check(e, "sticky CUDA error before tn_build_bs_unitary");
  cudaStream_t s = (cudaStream_t)stream;
  // K2 reads the plan's binomial table, uploaded asynchronously on the plan stream
  tn_status st = wait_tables(p, s);
  if (st != TN_OK) return st;
  st = cuda_check(cudaEventRecord(p->ev[2], s), "event");
  if (st != TN_OK) return st;
  st = cuda_check(launch_bs_unitary(p->d, p->N, theta, phi, p->d_binom, reinterpret_cast<double2*>(U_out), s),
                  "K2 launch");
  if (st != TN_OK) return st;
  st = cuda_check(cudaEventRecord(p->ev[3], s), "event");
  p->rec_k2 = st == TN_OK;
  if (st == TN_OK) st = cuda_check(plan_touch(p, s), "plan fence");
  return st;
}

}  // extern "C"

namespace tn {
// tn_theta_exec with an explicit A-row gather list (tn_theta_exec_sharded's slab scatter passes its own)
tn_status exec_impl(const tn_plan* p, tn_stream stream, const double* gamma_k, const double* lambda_k,
                    const double* gamma_k1, const double* lambda_l, const double* lambda_r, const double* U,
                    double* const* theta_out, const int32_t* rowperm) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_theta_exec: NULL plan");
  if (!gamma_k || !lambda_k || !gamma_k1 || !lambda_l || !lambda_r || !U || !theta_out)
    return fail(TN_ERR_DIMENSION, "tn_theta_exec: NULL input pointer");
  for (int c = 0; c < p->nsec; ++c)
    if (p->lR[c] * p->C[c] > 0 && !theta_out[c])
      return fail(TN_ERR_DIMENSION, "tn_theta_exec: NULL theta_out[c] for a non-empty sector");
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_check(e, "sticky CUDA error before tn_theta_exec");
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  p->rec_exec = true;  // the workspace is in use from here on (pool release fence)
  tn_status st = wait_tables(p, s);
  if (st != TN_OK) return st;
  SectorParams sp;
  if ((st = make_sector_params(p, theta_out, nullptr, 0, s, &sp)) != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[4], s), "event")) != TN_OK) return st;
  if (p->contraction == TN_CONTRACT_PAPER_LITERAL) {  // ablation: K3L → K4L, no K5
    st = cuda_check(launch_literal(p, sp, reinterpret_cast<const double2*>(gamma_k), lambda_k,
                                   reinterpret_cast<const double2*>(gamma_k1), lambda_l, lambda_r,
                                   reinterpret_cast<const double2*>(U), s, p->ev[5]),
                    "literal launch");
    if (st != TN_OK) return st;
    if ((st = cuda_check(cudaEventRecord(p->ev[6], s), "event")) != TN_OK) return st;
    if ((st = cuda_check(cudaEventRecord(p->ev[7], s), "event")) != TN_OK) return st;
    return cuda_check(plan_touch(p, s), "plan fence");
  }
  const bool emu = p->contraction == TN_CONTRACT_INT8_OZAKI;
  st = cuda_check(emu ? launch_oz_stage(p, reinterpret_cast<const double2*>(gamma_k), lambda_k,
                                        reinterpret_cast<const double2*>(gamma_k1), s, rowperm)
                      : launch_stage(p, reinterpret_cast<const double2*>(gamma_k), lambda_k,
                                     reinterpret_cast<const double2*>(gamma_k1), s, rowperm),
                  "K3 launch");
  if (st != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[5], s), "event")) != TN_OK) return st;
  if (p->pair) {  // MPO pair plan: K4 (or K4O), then the two-pass U⊗U* mix (tn_pair.cu)
    st = cuda_check(emu ? launch_oz_contract(p, sp, s) : launch_contract(p, sp, s), "K4 launch");
    if (st != TN_OK) return st;
    if ((st = cuda_check(cudaEventRecord(p->ev[6], s), "event")) != TN_OK) return st;
    st = cuda_check(launch_pair_mix(p, sp, lambda_l, lambda_r, reinterpret_cast<const double2*>(U), s), "K5P launch");
    if (st != TN_OK) return st;
  } else {
    st = cuda_check(emu ? launch_oz_contract(p, sp, s) : launch_contract(p, sp, s), "K4 launch");
    if (st != TN_OK) return st;
    if ((st = cuda_check(cudaEventRecord(p->ev[6], s), "event")) != TN_OK) return st;
    st = cuda_check(launch_mix(p, sp, lambda_l, lambda_r, reinterpret_cast<const double2*>(U), s), "K5 launch");
    if (st != TN_OK) return st;
  }
  if ((st = cuda_check(cudaEventRecord(p->ev[7], s), "event")) != TN_OK) return st;
  return cuda_check(plan_touch(p, s), "plan fence");
}
}  // namespace tn

extern "C" {

tn_status tn_theta_exec(const tn_plan* p, tn_stream stream, const double* gamma_k, const double* lambda_k,
                        const double* gamma_k1, const double* lambda_l, const double* lambda_r, const double* U,
                        double* const* theta_out) {
  return exec_impl(p, stream, gamma_k, lambda_k, gamma_k1, lambda_l, lambda_r, U, theta_out,
                   p ? p->d_rowperm : nullptr);
}

tn_status tn_theta_exec_remote(tn_plan* p, tn_stream stream, const double* gamma_k, const double* lambda_k,
                               const double* gamma_k1, const double* lambda_l, const double* lambda_r, const double* U,
                               double* const* theta_dst) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_theta_exec_remote: NULL plan");
  if (p->contraction == TN_CONTRACT_PAPER_LITERAL)
    return fail(TN_ERR_UNSUPPORTED, "tn_theta_exec_remote: the DMMA or INT8 engine only");
  if (!gamma_k || !lambda_k || !gamma_k1 || !lambda_l || !lambda_r || !U || !theta_dst)
    return fail(TN_ERR_DIMENSION, "tn_theta_exec_remote: NULL input pointer");
  for (int c = 0; c < p->nsec; ++c)
    if (p->lR[c] * p->C[c] > 0 && !theta_dst[c])
      return fail(TN_ERR_DIMENSION, "tn_theta_exec_remote: NULL theta_dst[c] for a non-empty slab");
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_check(e, "sticky CUDA error before tn_theta_exec_remote");
  // local P workspace of this rank's slab shapes (pooled, kept by the plan)
  std::vector<double*> pw(p->nsec, nullptr);
  {
    int64_t tot = 0;
    std::vector<int64_t> off(p->nsec, 0);
    for (int c = 0; c < p->nsec; ++c) {
      off[c] = tot;
      tot += (p->lR[c] * p->C[c] + 15) / 16 * 16;
    }
    if (!p->blk_p && tot > 0) {
      cudaError_t aerr = cudaSuccess;
      p->blk_p = pool_alloc((size_t)tot * sizeof(double2), &aerr);
      if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (remote P workspace)");
      p->ws_bytes += tot * (int64_t)sizeof(double2);
    }
    for (int c = 0; c < p->nsec; ++c)
      if (p->lR[c] * p->C[c] > 0) pw[c] = reinterpret_cast<double*>(static_cast<double2*>(p->blk_p) + off[c]);
  }
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  p->rec_exec = true;
  tn_status st = wait_tables(p, s);
  if (st != TN_OK) return st;
  SectorParams sp4, sp5;
  // K4 writes P into the local workspace (table 0); K5 reads it there and writes Θ to theta_dst (table 1)
  if ((st = make_sector_params(p, pw.data(), nullptr, 0, s, &sp4)) != TN_OK) return st;
  if ((st = make_sector_params(p, theta_dst, pw.data(), 1, s, &sp5)) != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[4], s), "event")) != TN_OK) return st;
  const bool emu = p->contraction == TN_CONTRACT_INT8_OZAKI;
  st = cuda_check(emu ? launch_oz_stage(p, reinterpret_cast<const double2*>(gamma_k), lambda_k,
                                        reinterpret_cast<const double2*>(gamma_k1), s, p->d_rowperm)
                      : launch_stage(p, reinterpret_cast<const double2*>(gamma_k), lambda_k,
                                     reinterpret_cast<const double2*>(gamma_k1), s, p->d_rowperm),
                  "K3 launch");
  if (st != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[5], s), "event")) != TN_OK) return st;
  st = cuda_check(emu ? launch_oz_contract(p, sp4, s) : launch_contract(p, sp4, s), "K4 launch");
  if (st != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[6], s), "event")) != TN_OK) return st;
  if (p->pair)  // K5P: pass 1 in place on the local workspace, pass 2 from it into the destination buffers
    st = cuda_check(launch_pair_mix(p, sp4, lambda_l, lambda_r, reinterpret_cast<const double2*>(U), s, &sp5),
                    "K5P launch");
  else
    st = cuda_check(launch_mix(p, sp5, lambda_l, lambda_r, reinterpret_cast<const double2*>(U), s), "K5 launch");
  if (st != TN_OK) return st;
  if ((st = cuda_check(cudaEventRecord(p->ev[7], s), "event")) != TN_OK) return st;
  return cuda_check(plan_touch(p, s), "plan fence");
}

// ---- CUDA IPC helpers: export a device buffer to another process, open a peer's buffer ----
tn_status tn_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(TN_ERR_DIMENSION, "tn_ipc_get_handle: NULL");
  // the allocation base via the driver API, resolved at run time (the library must load without a GPU)
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<GetRange>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!get_range) return fail(TN_ERR_CUDA, "tn_ipc_get_handle: libcuda.so.1 / cuMemGetAddressRange_v2 unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
    return fail(TN_ERR_CUDA, "tn_ipc_get_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  tn_status st = cuda_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  if (st != TN_OK) return st;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((unsigned long long)(uintptr_t)dev_ptr - base);
  return TN_OK;
}

tn_status tn_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(TN_ERR_DIMENSION, "tn_ipc_open: NULL");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  return cuda_check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

tn_status tn_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return TN_OK;
  return cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

}  // extern "C"
