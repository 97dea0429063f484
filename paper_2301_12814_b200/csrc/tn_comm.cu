// Row-sharded Θ exec over NCCL ("High-level parallelization"; BASELINE.json
// north_star: "partitioned across the 8 B200s of one box by sharding the α_{k-1} rows of Θ, with
// Γ^{[k+1]}, λ and U replicated; NCCL is used only to gather the shards or broadcast the operands").
//
// The compute needs no collective: each rank runs K3→K4→K5 on its flop-balanced row shard
// (tn_theta_plan(world_size, rank)). The exchange steps are
//  * the optional operand distribution from rank 0: Γk as ROW SLABS (each rank receives only its rows,
//    packed in sorted order by K6 `k6_pack_rows` on rank 0 and sent point to point — NCCL has no
//    scatterv), Γk1, λk, λl, λr and U by ncclBroadcast (they are replicated, north_star); or the whole
//    Γk broadcast (TN_BCAST_FULL, kept for comparison);
//  * the optional gather of every rank's Θ slabs to rank 0 (TN_GATHER_ROOT) or to each sector's owner
//    (TN_GATHER_SECTOR_OWNER), grouped ncclSend/ncclRecv that execute the transfer list
//    tn_plan_gather_schedule returns — the same list the host-only tn_gather_schedule_host computes,
//    which the multi-process gloo tests execute.
// NCCL is resolved at run time with dlopen so the library loads (and its single-GPU path runs) without
// it; torch's bundled libnccl.so.2 is normally already resident. After every grouped call the
// communicator's asynchronous error state is checked (ncclCommGetAsyncError).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

#include "nccl.h"
#include "tn_internal.cuh"

struct tn_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

namespace tn {
namespace {

struct NcclApi {
  bool loaded = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* env = std::getenv("TN_NCCL_LIB");
  void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define TN_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
  TN_SYM(GetUniqueId, "ncclGetUniqueId");
  TN_SYM(CommInitRank, "ncclCommInitRank");
  TN_SYM(CommDestroy, "ncclCommDestroy");
  TN_SYM(Broadcast, "ncclBroadcast");
  TN_SYM(Send, "ncclSend");
  TN_SYM(Recv, "ncclRecv");
  TN_SYM(GroupStart, "ncclGroupStart");
  TN_SYM(GroupEnd, "ncclGroupEnd");
  TN_SYM(GetErrorString, "ncclGetErrorString");
  TN_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef TN_SYM
  api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.Send && api.Recv &&
               api.GroupStart && api.GroupEnd && api.GetErrorString && api.CommGetAsyncError;
  return api;
}

tn_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return TN_OK;
  return fail(TN_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// The communicator's asynchronous error state (a peer failure or a network error surfaces here, not in the
// return code of the enqueueing call): ncclInProgress only means a non-blocking operation is still running.
tn_status async_check(ncclComm_t comm, const char* what) {
  ncclResult_t ae = ncclSuccess;
  ncclResult_t r = nccl().CommGetAsyncError(comm, &ae);
  if (r != ncclSuccess) return nccl_check(r, "ncclCommGetAsyncError");
  if (ae == ncclSuccess || ae == ncclInProgress) return TN_OK;
  return fail(TN_ERR_NCCL, std::string(what) + ": asynchronous NCCL error: " + nccl().GetErrorString(ae));
}

// K6 — rank 0 packs Γk's rows into sorted-position order, so every rank's slab [r0, r1) is one contiguous
// run to send: out[p − p0][:] = Γk[perm_l[p]][:] for p ∈ [p0, p1). HBM-bound copy, 16-B elements.
__global__ void __launch_bounds__(256) k6_pack_rows(const double2* __restrict__ gk, const int32_t* __restrict__ perm_l,
                                                    int64_t p0, int64_t rows, int64_t ld, double2* __restrict__ out) {
  const int64_t total = rows * ld;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ld, k = e - r * ld;
    out[e] = gk[(int64_t)perm_l[p0 + r] * ld + k];
  }
}

// The A-row gather list re-expressed as rows of this rank's packed slab: entry j = (sorted position of the
// row) − r0 (single-charge plans: positions are the identity; pair plans: the plan's d_rowpos).
__global__ void __launch_bounds__(256) k6_slab_rowlist(const int32_t* __restrict__ pos, int64_t n, int64_t r0,
                                                       int64_t r1, int32_t* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = pos ? pos[j] : j;
    out[j] = (q >= r0 && q < r1) ? (int32_t)(q - r0) : 0;  // rows outside the shard are never read
  }
}

// ---- the gather schedule (host logic shared by the plan call, the host-only call and the exec) ----
struct Transfer {
  int64_t sector, src, dst, row_begin, rows, cols;
};
static_assert(sizeof(Transfer) == sizeof(tn_transfer), "tn_transfer layout");

// rows_before(c, pos): rows of Θ(c) whose sorted left position is < pos; dest(c): receiving rank
template <class RowsBefore, class Dest>
void build_schedule(int nsec, const std::vector<int64_t>& C, const std::vector<int64_t>& bounds, RowsBefore rows_before,
                    Dest dest, std::vector<Transfer>& out) {
  out.clear();
  const int world = (int)bounds.size() - 1;
  for (int c = 0; c < nsec; ++c) {
    if (C[c] <= 0) continue;
    for (int src = 0; src < world; ++src) {
      const int64_t b = rows_before(c, bounds[src]), e = rows_before(c, bounds[src + 1]);
      if (e > b) out.push_back(Transfer{c, src, dest(c), b, e - b, C[c]});
    }
  }
}

}  // namespace

// Rows of Θ(c) whose sorted left position is < pos: its rows are [row0, row0+R) for single-charge plans,
// and for MPO pair plans whole left pair segments l = (l1, l2), l − (c1, c2) ∈ [0, d−1]², in key order
int64_t sector_rows_before(const tn_plan* p, int c, int64_t pos) {
  if (!p->pair) return std::min(std::max(pos, p->row0[c]), p->row0[c] + p->R[c]) - p->row0[c];
  const int nk = p->N + 1, c1 = c / nk, c2 = c % nk;
  const auto& ol = p->off[0];
  int64_t n = 0;
  for (int l1 = c1; l1 <= std::min(p->N, c1 + p->d - 1); ++l1)
    for (int l2 = c2; l2 <= std::min(p->N, c2 + p->d - 1); ++l2) {
      const int l = l1 * nk + l2;
      n += std::min<int64_t>(std::max<int64_t>(pos - ol[l], 0), (int64_t)ol[l + 1] - ol[l]);
    }
  return n;
}

static void plan_schedule(const tn_plan* p, int gather_mode, std::vector<Transfer>& out) {
  out.clear();
  if (gather_mode == TN_GATHER_NONE) return;
  build_schedule(
      p->nsec, p->C, p->bounds, [&](int c, int64_t pos) { return sector_rows_before(p, c, pos); },
      [&](int c) { return gather_mode == TN_GATHER_ROOT ? 0 : (p->owner.empty() ? 0 : p->owner[c]); }, out);
}

}  // namespace tn

using namespace tn;

extern "C" {

tn_status tn_comm_unique_id(void* id128) {
  if (!id128) return fail(TN_ERR_DIMENSION, "tn_comm_unique_id: NULL");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TN_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  ncclUniqueId id;
  tn_status st = nccl_check(api.GetUniqueId(&id), "ncclGetUniqueId");
  if (st == TN_OK) std::memcpy(id128, &id, sizeof(id));
  return st;
}

tn_status tn_comm_init(const void* id128, int rank, int world_size, tn_comm** out) {
  if (!id128 || !out) return fail(TN_ERR_DIMENSION, "tn_comm_init: NULL");
  *out = nullptr;
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(TN_ERR_DOMAIN, "tn_comm_init: bad rank/world");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TN_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  tn_comm* c = new (std::nothrow) tn_comm();
  if (!c) return fail(TN_ERR_OOM, "tn_comm_init: host allocation");
  tn_status st = nccl_check(api.CommInitRank(&c->comm, world_size, id, rank), "ncclCommInitRank");
  if (st != TN_OK) {
    delete c;
    return st;
  }
  c->rank = rank;
  c->world = world_size;
  *out = c;
  return TN_OK;
}

tn_status tn_comm_destroy(tn_comm* comm) {
  if (!comm) return TN_OK;
  tn_status st = TN_OK;
  if (comm->comm) st = nccl_check(nccl().CommDestroy(comm->comm), "ncclCommDestroy");
  delete comm;
  return st;
}

tn_status tn_comm_async_error(tn_comm* comm) {
  if (!comm) return fail(TN_ERR_DIMENSION, "tn_comm_async_error: NULL");
  if (!comm->comm) return TN_OK;
  return async_check(comm->comm, "tn_comm_async_error");
}

tn_status tn_plan_slab_rows(const tn_plan* p, int c, int rank, int64_t* row_begin, int64_t* rows) {
  if (!p || !row_begin || !rows) return fail(TN_ERR_DIMENSION, "tn_plan_slab_rows: NULL");
  if (c < 0 || c >= p->nsec) return fail(TN_ERR_DOMAIN, "tn_plan_slab_rows: sector out of range");
  if (rank < 0 || rank >= p->world) return fail(TN_ERR_DOMAIN, "tn_plan_slab_rows: rank out of range");
  const int64_t b = sector_rows_before(p, c, p->bounds[rank]), e = sector_rows_before(p, c, p->bounds[rank + 1]);
  *row_begin = b;
  *rows = e - b;
  return TN_OK;
}

static tn_status emit(const std::vector<Transfer>& v, int64_t capacity, tn_transfer* out, int64_t* n_out) {
  *n_out = (int64_t)v.size();
  if (out && capacity > 0) std::memcpy(out, v.data(), (size_t)std::min<int64_t>(capacity, *n_out) * sizeof(Transfer));
  if (out && capacity < *n_out) return fail(TN_ERR_DIMENSION, "gather schedule: capacity below the entry count");
  return TN_OK;
}

tn_status tn_plan_gather_schedule(const tn_plan* p, int gather_mode, int64_t capacity, tn_transfer* out,
                                  int64_t* n_out) {
  if (!p || !n_out) return fail(TN_ERR_DIMENSION, "tn_plan_gather_schedule: NULL");
  if (gather_mode != TN_GATHER_NONE && gather_mode != TN_GATHER_ROOT && gather_mode != TN_GATHER_SECTOR_OWNER)
    return fail(TN_ERR_DOMAIN, "tn_plan_gather_schedule: unknown gather_mode");
  std::vector<Transfer> v;
  plan_schedule(p, gather_mode, v);
  return emit(v, capacity, out, n_out);
}

tn_status tn_gather_schedule_host(int d, int N, const int32_t* off_l, const int32_t* off_r, int world_size,
                                  const int64_t* bounds, int gather_mode, int64_t capacity, tn_transfer* out,
                                  int64_t* n_out) {
  if (!off_l || !off_r || !bounds || !n_out) return fail(TN_ERR_DIMENSION, "tn_gather_schedule_host: NULL");
  if (d < 2 || N < 0 || N > TN_MAX_N || world_size < 1) return fail(TN_ERR_DOMAIN, "tn_gather_schedule_host: bad d/N/world");
  if (gather_mode != TN_GATHER_NONE && gather_mode != TN_GATHER_ROOT && gather_mode != TN_GATHER_SECTOR_OWNER)
    return fail(TN_ERR_DOMAIN, "tn_gather_schedule_host: unknown gather_mode");
  for (int q = 0; q <= N; ++q)
    if (off_l[q + 1] < off_l[q] || off_r[q + 1] < off_r[q]) return fail(TN_ERR_DOMAIN, "tn_gather_schedule_host: offsets decrease");
  for (int r = 0; r < world_size; ++r)
    if (bounds[r + 1] < bounds[r]) return fail(TN_ERR_DOMAIN, "tn_gather_schedule_host: bounds decrease");
  // sectors exactly as tn_theta_plan lays them out (R2)
  std::vector<int64_t> R(N + 1), C(N + 1), row0(N + 1), sizes(N + 1);
  for (int c = 0; c <= N; ++c) {
    row0[c] = off_l[c];
    R[c] = off_l[std::min(N, c + d - 1) + 1] - off_l[c];
    C[c] = off_r[c + 1] - off_r[std::max(0, c - d + 1)];
    sizes[c] = R[c] * C[c];
  }
  std::vector<int32_t> owner;
  sector_owners(sizes, world_size, owner);
  std::vector<int64_t> b(bounds, bounds + world_size + 1);
  std::vector<Transfer> v;
  if (gather_mode != TN_GATHER_NONE)
    build_schedule(
        N + 1, C, b, [&](int c, int64_t pos) { return std::min(std::max(pos, row0[c]), row0[c] + R[c]) - row0[c]; },
        [&](int c) { return gather_mode == TN_GATHER_ROOT ? 0 : owner[c]; }, v);
  return emit(v, capacity, out, n_out);
}

static tn_status ensure_slab_rowlist(const tn_plan* p, cudaStream_t s) {
  if (p->blk_slab) return TN_OK;
  cudaError_t aerr = cudaSuccess;
  tn_plan* pm = const_cast<tn_plan*>(p);
  pm->blk_slab = pool_alloc((size_t)std::max<int64_t>(1, p->n_rowlist) * sizeof(int32_t), &aerr);
  if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (slab row list)");
  pm->d_slab_rowlist = static_cast<int32_t*>(pm->blk_slab);
  if (p->n_rowlist == 0) return TN_OK;
  tn_status st = cuda_check(cudaStreamWaitEvent(s, p->ev_ready, 0), "wait for plan tables");
  if (st != TN_OK) return st;
  const unsigned grid = (unsigned)std::min<int64_t>((p->n_rowlist + 255) / 256, 1024);
  k6_slab_rowlist<<<grid, 256, 0, s>>>(p->d_rowpos, p->n_rowlist, p->r0, p->r1, pm->d_slab_rowlist);
  return cuda_check(cudaGetLastError(), "K6 slab row list");
}

static tn_status pack_rows(const tn_plan* p, cudaStream_t s, const double* gamma_k, int64_t p0, int64_t p1, double* out) {
  const int64_t rows = p1 - p0, chi_c = p->chi[1];
  if (rows <= 0) return TN_OK;
  tn_status st = cuda_check(cudaStreamWaitEvent(s, p->ev_ready, 0), "wait for plan tables");
  if (st != TN_OK) return st;
  const unsigned grid = (unsigned)std::min<int64_t>((rows * chi_c + 255) / 256, (int64_t)p->sm_count * 16);
  k6_pack_rows<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(gamma_k), p->d_perm[0], p0, rows, chi_c,
                                    reinterpret_cast<double2*>(out));
  if ((st = cuda_check(cudaGetLastError(), "K6 pack rows")) != TN_OK) return st;
  return cuda_check(plan_touch(p, s), "plan fence");
}

tn_status tn_pack_row_slab(const tn_plan* p, tn_stream stream, const double* gamma_k, int rank, double* slab_out) {
  if (!p || !gamma_k || !slab_out) return fail(TN_ERR_DIMENSION, "tn_pack_row_slab: NULL");
  if (rank < 0 || rank >= p->world) return fail(TN_ERR_DOMAIN, "tn_pack_row_slab: rank outside [0, world)");
  return pack_rows(p, (cudaStream_t)stream, gamma_k, p->bounds[rank], p->bounds[rank + 1], slab_out);
}

tn_status tn_theta_exec_slab(const tn_plan* p, tn_stream stream, const double* gamma_k_slab, const double* lambda_k,
                             const double* gamma_k1, const double* lambda_l, const double* lambda_r, const double* U,
                             double* const* theta_out) {
  if (!p) return fail(TN_ERR_DIMENSION, "tn_theta_exec_slab: NULL plan");
  if (p->contraction == TN_CONTRACT_PAPER_LITERAL)
    return fail(TN_ERR_UNSUPPORTED, "tn_theta_exec_slab: the literal ablation engine reads Γk in caller order");
  tn_status st = ensure_slab_rowlist(p, (cudaStream_t)stream);
  if (st != TN_OK) return st;
  return exec_impl(p, stream, gamma_k_slab, lambda_k, gamma_k1, lambda_l, lambda_r, U, theta_out, p->d_slab_rowlist);
}

tn_status tn_theta_exec_sharded(const tn_plan* p, tn_stream stream, tn_comm* comm, double* gamma_k,
                                double* lambda_k, double* gamma_k1, double* lambda_l, double* lambda_r, double* U,
                                double* const* theta_out, int bcast_operands, int gather_mode) {
  if (!p || !comm) return fail(TN_ERR_DIMENSION, "tn_theta_exec_sharded: NULL plan/comm");
  if (p->world != comm->world || p->rank != comm->rank)
    return fail(TN_ERR_CONSISTENCY, "tn_theta_exec_sharded: plan world/rank differ from the communicator's");
  if (gather_mode != TN_GATHER_NONE && gather_mode != TN_GATHER_ROOT && gather_mode != TN_GATHER_SECTOR_OWNER)
    return fail(TN_ERR_DOMAIN, "tn_theta_exec_sharded: unknown gather_mode");
  if (bcast_operands != TN_BCAST_NONE && bcast_operands != TN_BCAST_SLABS && bcast_operands != TN_BCAST_FULL)
    return fail(TN_ERR_DOMAIN, "tn_theta_exec_sharded: unknown bcast_operands mode");
  if (bcast_operands == TN_BCAST_SLABS && p->contraction == TN_CONTRACT_PAPER_LITERAL)
    return fail(TN_ERR_UNSUPPORTED, "tn_theta_exec_sharded: the literal ablation engine reads Γk in caller order (use TN_BCAST_FULL)");
  if (!theta_out) return fail(TN_ERR_DIMENSION, "tn_theta_exec_sharded: NULL theta_out");
  if (!gamma_k || !lambda_k || !gamma_k1 || !lambda_l || !lambda_r || !U)
    return fail(TN_ERR_DIMENSION, "tn_theta_exec_sharded: NULL input pointer");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TN_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  tn_status st = async_check(comm->comm, "before tn_theta_exec_sharded");
  if (st != TN_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t chi_l = p->chi[0], chi_c = p->chi[1];
  const int32_t* rowperm = p->d_rowperm;
  if (bcast_operands != TN_BCAST_NONE) {
    const bool slabs = bcast_operands == TN_BCAST_SLABS;
    double* pack = nullptr;
    if (slabs && p->rank == 0 && p->world > 1) {  // rank 0: the other ranks' rows in sorted order, one run each
      if (!p->blk_pack) {
        cudaError_t aerr = cudaSuccess;
        const_cast<tn_plan*>(p)->blk_pack = pool_alloc((size_t)(chi_l - p->bounds[1]) * chi_c * sizeof(double2) + 256, &aerr);
        if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (Γk slab staging)");
      }
      pack = static_cast<double*>(p->blk_pack);
      if ((st = pack_rows(p, s, gamma_k, p->bounds[1], chi_l, pack)) != TN_OK) return st;
    }
    if (slabs && p->rank != 0) {  // K3 reads the received packed slab through the plan's slab row list
      if ((st = ensure_slab_rowlist(p, s)) != TN_OK) return st;
      rowperm = p->d_slab_rowlist;
    }
    st = nccl_check(api.GroupStart(), "ncclGroupStart");
    if (st != TN_OK) return st;
    const size_t n_gk1 = (size_t)(2 * p->chi[1] * p->chi[2]);
    ncclResult_t r = ncclSuccess;
    if (slabs) {
      if (p->rank == 0) {
        for (int dst = 1; dst < p->world && r == ncclSuccess; ++dst) {
          const int64_t rows = p->bounds[dst + 1] - p->bounds[dst];
          if (rows > 0)
            r = api.Send(pack + 2 * (p->bounds[dst] - p->bounds[1]) * chi_c, (size_t)(2 * rows * chi_c), ncclFloat64, dst,
                         comm->comm, s);
        }
      } else if (p->r1 > p->r0) {
        r = api.Recv(gamma_k, (size_t)(2 * (p->r1 - p->r0) * chi_c), ncclFloat64, 0, comm->comm, s);
      }
    } else {
      r = api.Broadcast(gamma_k, gamma_k, (size_t)(2 * chi_l * chi_c), ncclFloat64, 0, comm->comm, s);
    }
    if (r == ncclSuccess) r = api.Broadcast(gamma_k1, gamma_k1, n_gk1, ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_k, lambda_k, (size_t)p->chi[1], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_l, lambda_l, (size_t)p->chi[0], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_r, lambda_r, (size_t)p->chi[2], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(U, U, (size_t)(2 * p->u_size), ncclFloat64, 0, comm->comm, s);
    ncclResult_t r2 = api.GroupEnd();
    st = nccl_check(r != ncclSuccess ? r : r2, slabs ? "operand distribution (Γk slabs + broadcasts)" : "operand broadcast");
    if (st == TN_OK) st = async_check(comm->comm, "operand distribution");
    if (st != TN_OK) return st;
  }
  std::vector<Transfer> sched;
  plan_schedule(p, gather_mode, sched);
  // Local slabs: where this rank receives a whole sector (ROOT: rank 0, SECTOR_OWNER: the sector's owner) the
  // caller passed the FULL Θ(c), and this rank's slab is written in place at its schedule row.
  std::vector<double*> local(p->nsec, nullptr);
  for (int c = 0; c < p->nsec; ++c) local[c] = theta_out[c];
  for (const Transfer& t : sched)
    if (t.src == p->rank && t.dst == p->rank && theta_out[t.sector])
      local[t.sector] = theta_out[t.sector] + 2 * t.row_begin * t.cols;
  st = exec_impl(p, stream, gamma_k, lambda_k, gamma_k1, lambda_l, lambda_r, U, local.data(), rowperm);
  if (st != TN_OK || gather_mode == TN_GATHER_NONE) return st;
  st = nccl_check(api.GroupStart(), "ncclGroupStart");
  if (st != TN_OK) return st;
  ncclResult_t r = ncclSuccess;
  for (const Transfer& t : sched) {
    if (r != ncclSuccess) break;
    if (t.src == t.dst) continue;  // written in place above
    const size_t n = (size_t)(2 * t.rows * t.cols);
    if (t.dst == p->rank)
      r = api.Recv(theta_out[t.sector] + 2 * t.row_begin * t.cols, n, ncclFloat64, (int)t.src, comm->comm, s);
    else if (t.src == p->rank)
      r = api.Send(theta_out[t.sector], n, ncclFloat64, (int)t.dst, comm->comm, s);
  }
  ncclResult_t r2 = api.GroupEnd();
  st = nccl_check(r != ncclSuccess ? r : r2, gather_mode == TN_GATHER_ROOT ? "Θ gather to root" : "Θ gather to sector owners");
  if (st == TN_OK) st = async_check(comm->comm, "Θ gather");
  return st;
}

}  // extern "C"
