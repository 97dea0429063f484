// Internal declarations shared by the kernels and the C-ABI glue of libtn_theta.so (product path).
// Nothing here is shared with oracle/ (the two share no code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/tn_theta.h"

namespace tn {

// ---------------------------------------------------------------------------------------------
// Tiling constants of the K4 contraction (DESIGN.md §4 "K4").
//   CTA tile BM×BN complex outputs, 8 consumer warps in 2×4, each 32×16 = 4×2 DMMA.8x8x4 tiles.
//   K is consumed in chunks of BK; the chunk is one cp.async.bulk (TMA 1-D) copy per operand.
// ---------------------------------------------------------------------------------------------
constexpr int BM = 64;
constexpr int BN = 64;
constexpr int BK = 16;
constexpr int CHUNK = BM * BK;        // complex elements per full operand chunk (== BN * BK)
constexpr int K4_STAGES = 6;
constexpr int K4_CONSUMER_WARPS = 8;
constexpr int K4_THREADS = (K4_CONSUMER_WARPS + 1) * 32;

struct GroupDesc {          // one center charge c_c: P_{c_c} = A_{c_c} · B_{c_c}
  int64_t a_off;            // complex offset of this group's A panel in the A workspace
  int64_t b_off;            // complex offset of this group's B panel in the B workspace
  int64_t row0;             // first sorted left position of the group's (local) rows
  int64_t col0;             // first sorted right position of the group's columns
  int64_t k0;               // first sorted center position of seg_c(c_c)
  int32_t R, C, K, K4;      // local rows, cols, true K, K padded to a multiple of 4
  int32_t cc;               // the center charge == the output sector written with P
  int32_t nmt, nnt, pad;
};

struct TileDesc {
  int32_t g, mt, nt, pad;
};

struct LitSector {          // paper-literal ablation (k4l_literal.cu): one Θ(c) as one GEMM
  int64_t a_off, b_off;     // complex offsets of its A / B panels
  int64_t row0, col0;       // sorted positions of its first (local) row / column
  int32_t c, R, C, K4;      // sector, local rows, cols, padded K (segments rounded up to BK)
  int32_t nmt, nnt, seg0, nseg;  // tiles; its centre segments in the segment table
};

struct MixTile2 {           // K5P work unit (pair plans): one species' U mix over ≤ ~128 8-groups of one (l, r) block
  int32_t cl, n, lo, L;     // that species' left charge, U block n = l_s − r_s, first index lo, vector length L
  int32_t e0, ne, nr, ngr;  // as MixTile (8-groups row-major over the tile's rows of segment l)
  int32_t pl0, pr0;         // sorted positions of the tile's first row / the block's first column
  int32_t lkey, rkey;       // pair keys of the left / right segment
  int32_t fixed, band;      // the other species' output value; the tile's first row within segment l
  int32_t flags, nfix;      // bit 0: pass 2 (species 2: conj(U), sectors (fixed, lo+u), outer λ's); values fixed..+nfix−1
};

struct MixTile {            // K5 work unit: ≤ 128 "8-groups" (8 consecutive columns of one row) of one (c_l, c_r) block
  int32_t cl, cr;           // left / right charge
  int32_t e0, ne;           // first 8-group (row-major within the block) and count
  int32_t nr, ngr;          // columns of the block (n_r(c_r)) and 8-groups per row ⌈nr/8⌉
  int32_t pl0, pr0;         // sorted positions of the block's first (local) row / first column
};

constexpr int MAXC = TN_MAX_N + 1;

// ---------------------------------------------------------------------------------------------
// INT8 tensor-core emulation of the FP64 contraction (Ozaki splitting; DESIGN.md §4 "K3O/K4O").
//   Tile: OZ_BM rows × OZ_BN columns of one group, K consumed in OZ_BK-byte steps (one UMMA K).
//   A (R×K) and B (K×C) are split into S signed 7-bit slices with per-row / per-column power-of-two
//   scales; slice products accumulate exactly in int32 TMEM, one accumulator per diagonal p+q.
// ---------------------------------------------------------------------------------------------
constexpr int OZ_BM = 128;
constexpr int OZ_BN = 64;
constexpr int OZ_BK = 32;
constexpr int OZ_SMIN = 4, OZ_SMAX = 8;
constexpr int OZ_KMAX = 2048;             // largest centre segment the INT8 emulation accepts
constexpr int OZ_A_TILE = OZ_BM * OZ_BK;  // bytes of one A slice tile (canonical K-major layout)
constexpr int OZ_B_TILE = OZ_BN * OZ_BK;  // bytes of one B slice tile

struct OzGroup {
  int64_t a_off, b_off;     // byte offsets of this group's A / B slice tiles
  int64_t ea_off, eb_off;   // offsets of its row / column exponents (int32)
  int64_t row0, col0, k0;   // sorted positions of the first row / column / center bond
  int32_t R, C, K, Kp;      // local rows, cols, K, K padded to OZ_BK
  int32_t nmt, nnt, nkc, cc;
};
struct OzTile {
  int32_t g, mt, nt, pad;
};

// Per-sector table in device memory (DESIGN.md §4 "Runtime pieces"): the static part (slab origin, ld, whether
// the centre segment of that key is non-empty) is uploaded with the plan; the caller's output pointers (and
// the P source of tn_theta_exec_remote) are written by k_set_sectors at the start of every exec, so the table
// size is not limited by the kernel-parameter space and an exec stays capturable into a CUDA graph.
constexpr int MAX_SEC = 1024;   // sectors / charge keys of one plan: N+1 ≤ 101; pair plans (N+1)² ≤ 1024 (N ≤ 31)
struct SecEntry {
  double2* out;             // this rank's slab of Θ(c) (row-major, ld = C_c)
  const double2* src;       // K5 reads P_{c_c} from here when set (tn_theta_exec_remote), else from out
  int64_t lrow0;            // sorted left position of slab row 0
  int64_t col0;             // sorted right position of column 0
  int32_t ld;               // C_c
  int32_t nonempty;         // seg_c(c) is non-empty (K4 ran group c: P_c exists), c read as a centre key
};
struct SectorParams {
  SecEntry* sec;            // device table, one entry per sector / key
  const int32_t* ustart;    // device packed-U block offsets
  int32_t d, N;
};
struct SectorPtrs {         // k_set_sectors' by-value argument (≤ 16 KB of the 32 KB kernel-parameter space)
  double2* out[MAX_SEC];
  const double2* src[MAX_SEC];
  int32_t n;
};

}  // namespace tn

struct tn_plan {
  int d = 0, N = 0, world = 1, rank = 0;
  bool pair = false;                           // MPO plan: two charge species, key = c1·(N+1) + c2
  int nq = 0;                                  // charge keys: N+1, or (N+1)² for pair plans
  int nsec = 0;                                // output sectors (= nq)
  int64_t chi[3] = {0, 0, 0};
  std::vector<int32_t> off[3];                 // host copies of the offset tables (N+2)
  int32_t* d_perm[3] = {nullptr, nullptr, nullptr};  // device perm (sorted pos -> caller index)
  int32_t* d_qs[3] = {nullptr, nullptr, nullptr};    // device sorted charges
  int32_t* d_off[3] = {nullptr, nullptr, nullptr};   // device offset tables (N+2)
  double2* d_binom = nullptr;                  // (nmax+1)² exact binomials as double-double (K2)
  tn::SecEntry* d_sec[2] = {nullptr, nullptr}; // sector tables: [0] exec / remote K4, [1] remote K5 (tn_theta_exec_remote)
  int32_t* d_ustart = nullptr;                 // packed-U block offsets (device)
  std::vector<tn::SecEntry> h_sec;             // static part of the sector table (host source of the upload)
  std::vector<int64_t> bounds;                 // world+1 shard bounds (sorted left positions)
  std::vector<int32_t> owner;                  // TN_GATHER_SECTOR_OWNER: receiving rank of every sector
  int64_t r0 = 0, r1 = 0;                      // this rank's window
  // sectors
  std::vector<int64_t> R, C, row0, col0, lR, lrow0;   // global + local slab
  // groups / tiles
  std::vector<tn::GroupDesc> groups;
  tn::GroupDesc* d_groups = nullptr;
  tn::TileDesc* d_tiles = nullptr;
  int64_t ntiles = 0;
  tn::MixTile* d_mix = nullptr;
  int64_t nmix = 0;                            // K5 tiles
  int64_t nmix_cls[3] = {0, 0, 0};             // of which the first [0] have L ≤ 8, the next [1] L ≤ 16, [2] L ≤ 32
  // row / column index lists K3 and K3O gather through: perm_l / perm_r themselves for single-charge
  // plans (group rows are contiguous sorted positions), per-group gathered lists for pair plans
  const int32_t* d_rowperm = nullptr;
  const int32_t* d_colperm = nullptr;
  const int32_t* d_rowpos = nullptr;           // pair plans: sorted left position of every d_rowperm entry (single: identity)
  int64_t n_rowlist = 0;                       // entries of d_rowperm (single-charge: χ_l)
  // tn_theta_exec_sharded's Γk slab scatter (TN_BCAST_SLABS): d_rowperm re-expressed as rows of this rank's
  // packed slab (sorted position − r0), and on rank 0 the staging copy of Γk in sorted row order
  void* blk_slab = nullptr;
  int32_t* d_slab_rowlist = nullptr;
  void* blk_pack = nullptr;
  // pair plans: two-pass U⊗U* mix (tn_pair.cu)
  tn::MixTile2* d_mix2 = nullptr;
  int32_t* d_rowoff = nullptr;                 // [sector][left key]: local row of the segment in the sector (−1: absent)
  int32_t* d_coloff = nullptr;                 // [sector][right key]: local column of the segment
  int64_t nmix2[2] = {0, 0};                   // tiles of pass 1 (species 1) and pass 2 (species 2)
  int nfix_max = 1;                            // most values of the other species one K5P tile covers
  int64_t nmix2_multi[2] = {0, 0};             // of each pass's tiles, the trailing ones covering > 1 value
  // tiles per (pass, single/multi-value, register class L ≤ 8 / ≤ 16 / ≤ 32 / larger), in that order in d_mix2
  int64_t nmix2_grp[2][2][4] = {};
  int64_t nmix_fused = 0;                      // K5F tiles (blocks with L1, L2 ≤ 8: both species in one pass), first in d_mix2
  std::vector<tn::MixTile2> h_mix2;
  std::vector<int32_t> h_rowoff, h_coloff;
  std::vector<int32_t> h_rowperm_pos, h_colperm_pos;
  void* blk_p = nullptr;                       // local P workspace of tn_theta_exec_remote (slab shapes)
  double2* d_apanel = nullptr;
  double2* d_bpanel = nullptr;
  int64_t a_elems = 0, b_elems = 0;
  int64_t u_size = 0;
  std::vector<int32_t> ustart;
  int64_t f_contract = 0, f_mix = 0, f_exec = 0, f_contract_local = 0, f_mix_local = 0;
  int64_t ws_bytes = 0;
  int max_mix = 0;                             // min(N+1, d): longest U-mix vector
  int sm_count = 148;
  cudaStream_t plan_stream = nullptr;
  int n_staged = 0;                            // ranges of the pinned upload ring not yet sealed (plan_h2d)
  void* blk_tab = nullptr;                     // pool block: perm / qs / off tables
  void* blk_work = nullptr;                    // pool block: group + tile tables, A/B panels
  // per-kernel timing events: [0,1] K1, [2,3] K2, [4] K3 start, [5] K4 start, [6] K5 start, [7] end
  cudaEvent_t ev[8] = {};
  // tables uploaded on plan_stream; exec waits for this event instead of the host syncing
  cudaEvent_t ev_ready = nullptr;
  std::vector<tn::TileDesc> h_tiles;           // host sources of the async uploads (kept alive)
  std::vector<tn::MixTile> h_mix;
  std::vector<tn::OzTile> h_oz_tiles;
  mutable bool rec_k1 = false, rec_k2 = false, rec_exec = false;
  mutable cudaStream_t last_stream = nullptr;  // stream of the last exec (pool release fence)
  mutable bool captured = false;               // an exec was captured into a CUDA graph (free_plan syncs the device)
  mutable cudaEvent_t ev_fence = nullptr;      // end of the last library work touching the plan's memory (pool fence)
  mutable cudaStream_t touch_stream = nullptr; // stream ev_fence was last recorded on
  mutable bool touch_stream_set = false;
  int dev = 0;
  // contraction mode (TN_CONTRACT_*) and the INT8-emulation layout (built by tn_plan_set_contraction)
  int contraction = TN_CONTRACT_F64_DMMA;
  int oz_slices = 0;
  std::vector<tn::OzGroup> oz_groups;
  tn::OzGroup* d_oz_groups = nullptr;
  tn::OzTile* d_oz_tiles = nullptr;
  int64_t oz_ntiles = 0;
  int8_t* d_oa = nullptr;
  int8_t* d_ob = nullptr;
  int32_t* d_oea = nullptr;
  int32_t* d_oeb = nullptr;
  void* blk_oz = nullptr;
  // paper-literal ablation engine (TN_CONTRACT_PAPER_LITERAL, k4l_literal.cu)
  std::vector<tn::LitSector> lit_secs;
  std::vector<tn::TileDesc> h_lit_tiles;
  std::vector<char> h_lit_segs;
  tn::LitSector* d_lit_secs = nullptr;
  void* d_lit_segs = nullptr;
  tn::TileDesc* d_lit_tiles = nullptr;
  double2* d_lit_a = nullptr;
  double2* d_lit_b = nullptr;
  int64_t lit_ntiles = 0, lit_flops = 0;
  void* blk_lit = nullptr;
  int64_t oz_macs = 0;                         // int8 MACs one exec issues
};

namespace tn {

inline cudaError_t plan_touch(const tn_plan* p, cudaStream_t s) {
  if (!p->ev_fence) return cudaSuccess;
  // one event covers every stream that touched the plan: a new stream first joins the previous fence
  if (p->touch_stream_set && p->touch_stream != s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
      cudaError_t e = cudaStreamWaitEvent(s, p->ev_fence, 0);
      if (e != cudaSuccess) return e;
    }
  }
  p->touch_stream = s;
  p->touch_stream_set = true;
  return cudaEventRecord(p->ev_fence, s);
}

void set_error(const std::string& s);
tn_status fail(tn_status st, const std::string& s);
tn_status cuda_check(cudaError_t e, const char* what);

// TN_GATHER_SECTOR_OWNER owners: LPT over element counts (tn_api.cu); rows of Θ(c) before a sorted left
// position (tn_comm.cu)
void sector_owners(const std::vector<int64_t>& sizes, int world, std::vector<int32_t>& owner);
int64_t sector_rows_before(const tn_plan* p, int c, int64_t pos);
// fill table `which` with the caller's output pointers (and P sources) on stream s; returns the kernel view
tn_status make_sector_params(const tn_plan* p, double* const* out, const double* const* src, int which,
                             cudaStream_t s, SectorParams* sp);
// make s wait for the plan's asynchronous table upload (host wait under graph capture)
tn_status wait_tables(const tn_plan* p, cudaStream_t s);
tn_status exec_impl(const tn_plan* p, tn_stream stream, const double* gamma_k, const double* lambda_k,
                    const double* gamma_k1, const double* lambda_l, const double* lambda_r, const double* U,
                    double* const* theta_out, const int32_t* rowperm);

// ---- kernel launchers (stream-ordered) ----
struct SortArgs {           // K1: one CTA per bond (0 = left, 1 = center, 2 = right)
  const int32_t* q[3];
  const int32_t* q2[3];     // second charge species (MPO pair plans; nullptr otherwise): key = q·(N+1) + q2
  int64_t chi[3];
  int32_t* perm[3];
  int32_t* qs[3];
  int32_t* off[3];
  int32_t* err;             // err[b] = 1 if a charge of bond b lies outside [0, N]
};
cudaError_t launch_sort_bonds(const SortArgs& a, int N, cudaStream_t s);
void* pool_alloc(size_t bytes, cudaError_t* err);
void pool_release(void* ptr, cudaStream_t last_stream, bool used);
cudaError_t pool_reserve_like(const void* ptr, int count);  // ≥ count blocks fitting ptr's request
// Shared fences: a destroyed plan hands its last-use event (recorded right after the last library work that
// touched its memory) to all of its blocks, so a block is reusable as soon as THAT work is done — not only once
// everything queued up to the destroy call has drained.
struct Fence {
  cudaEvent_t ev;
  int refs;
};
Fence* fence_adopt(cudaEvent_t ev);               // takes ownership of ev
void pool_release_fenced(void* ptr, Fence* f);    // the block shares f (nullptr: reusable at once)
void fence_release(Fence* f);                     // drop a fence no block adopted
// Plan shells: the plan's own stream and timing events are recycled between plans (stream creation costs
// tens of µs per gate otherwise).
struct PlanShell {
  int dev = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_ready = nullptr;
};
// Async H2D of a plan table on the plan stream, staged through the process-wide pinned ring (tn_pool.cu) when it
// fits: a pageable source costs the host a driver-side staging copy per call (measured 14–65 µs per phase of
// tn_theta_plan). plan_h2d_seal records the event that releases the plan's staged ranges (called after the
// plan's last upload, and again — harmlessly — when the plan is destroyed).
cudaError_t plan_h2d(tn_plan* p, void* dst, const void* src, size_t bytes);
// several host arrays into one device region [dst_base, dst_base + total): one staged copy (gaps undefined), or
// one pageable copy per part when the ring cannot take it
struct H2DPart {
  size_t off;
  const void* src;
  size_t bytes;
};
cudaError_t plan_h2d_parts(tn_plan* p, char* dst_base, const H2DPart* parts, int n, size_t total);
void plan_h2d_seal(tn_plan* p);
cudaError_t shell_acquire(PlanShell* out);
void shell_release(const PlanShell& sh);
// record the plan's pool fence at the current tail of s (after library work that touched the plan's memory)
inline cudaError_t plan_touch(const tn_plan* p, cudaStream_t s);
cudaError_t launch_bs_unitary(int d, int N, double theta, double phi, const double2* binom, double2* U,
                              cudaStream_t s);
// rowperm: the A-row gather list (p->d_rowperm; tn_theta_exec_sharded passes a slab list when Γk arrived as
// this rank's packed row slab)
cudaError_t launch_stage(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1,
                         cudaStream_t s, const int32_t* rowperm);
cudaError_t launch_contract(const tn_plan* p, const SectorParams& sp, cudaStream_t s);
cudaError_t launch_oz_stage(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1,
                            cudaStream_t s, const int32_t* rowperm);
cudaError_t launch_oz_contract(const tn_plan* p, const SectorParams& sp, cudaStream_t s);
// Per-thread auxiliary streams for launches that touch disjoint data (K3 a/b, K3O's two exponent→slice
// chains, K5's register classes): fork from s, run, join back into s. One set per (device, caller stream),
// so gates in flight on different caller streams of one thread share no auxiliary stream (no false
// cross-gate dependencies); a thread keeps at most AUX_SETS sets and recycles the least recently used one
// (reuse only adds ordering, never a hazard).
struct AuxStreams {
  int dev = -1;
  cudaStream_t owner = nullptr;  // the caller stream this set serves
  uint64_t used = 0;             // LRU stamp
  cudaStream_t st[3] = {};
  cudaEvent_t fork = nullptr, join[3] = {};
};
constexpr int AUX_SETS = 8;
inline cudaError_t aux_streams(cudaStream_t s, AuxStreams** out) {
  thread_local AuxStreams sets[AUX_SETS];
  thread_local uint64_t clock = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  AuxStreams* hit = nullptr;
  AuxStreams* lru = &sets[0];
  for (auto& a : sets) {
    if (a.dev == dev && a.owner == s) {
      hit = &a;
      break;
    }
    if (a.used < lru->used) lru = &a;
  }
  if (!hit) {
    hit = lru;
    if (hit->dev != dev) {  // (re)create on this device; release the old device's handles first
      if (hit->dev >= 0) {
        int cur = dev;
        cudaSetDevice(hit->dev);
        for (auto& x : hit->st) cudaStreamDestroy(x);
        cudaEventDestroy(hit->fork);
        for (auto& x : hit->join) cudaEventDestroy(x);
        cudaSetDevice(cur);
        hit->dev = -1;
      }
      for (auto& x : hit->st)
        if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&hit->fork, cudaEventDisableTiming)) != cudaSuccess) return e;
      for (auto& x : hit->join)
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
      hit->dev = dev;
    }
    hit->owner = s;
  }
  hit->used = ++clock;
  *out = hit;
  return cudaSuccess;
}

cudaError_t launch_mix(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                       const double2* U, cudaStream_t s, int first_class = 0);
void build_mix_tiles(tn_plan* p, std::vector<MixTile>& out);
tn_status build_pair_tables(tn_plan* p);
tn_status build_literal(tn_plan* p);
cudaError_t launch_literal(const tn_plan* p, const SectorParams& sp, const double2* gk, const double* lk,
                           const double2* gk1, const double* ll, const double* lr, const double2* U, cudaStream_t s,
                           cudaEvent_t mid);
cudaError_t launch_pair_mix(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                            const double2* U, cudaStream_t s, const SectorParams* sp2 = nullptr);

// ---- double-double arithmetic (K2): error-free transforms, ~106-bit significand ----
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_from(double a) { return {a, 0.0}; }
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  dd t = two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  p.lo = __fma_rn(x.hi, y.lo, p.lo);
  p.lo = __fma_rn(x.lo, y.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd x, dd y) {
  double q1 = x.hi / y.hi;
  dd r = dd_add(x, dd_neg(dd_mul(dd_from(q1), y)));
  double q2 = r.hi / y.hi;
  r = dd_add(r, dd_neg(dd_mul(dd_from(q2), y)));
  double q3 = r.hi / y.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd_from(q3));
}
__device__ __forceinline__ dd dd_sqrt(dd x) {
  if (x.hi <= 0.0) return {0.0, 0.0};
  double a = sqrt(x.hi);
  dd r = dd_add(x, dd_neg(two_prod(a, a)));
  return quick_two_sum(a, r.hi / (2.0 * a));
}

}  // namespace tn
