// Row-sharded Θ exec over NCCL ("High-level parallelization"; BASELINE.json
// north_star: "partitioned across the 8 B200s of one box by sharding the α_{k-1} rows of Θ, with
// Γ^{[k+1]}, λ and U replicated; NCCL is used only to gather the shards or broadcast the operands").
//
// The compute needs no collective: each rank runs K3→K4→K5 on its flop-balanced row shard
// (tn_theta_plan(world_size, rank)). The only exchange steps are the optional operand broadcast from
// rank 0 and the optional gather of every rank's Θ slabs to rank 0 (grouped ncclSend/ncclRecv,
// NCCL has no gatherv). NCCL is resolved at run time with dlopen so the library loads (and its
// single-GPU path runs) without it; torch's bundled libnccl.so.2 is normally already resident.
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
#undef TN_SYM
  api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.Send && api.Recv &&
               api.GroupStart && api.GroupEnd && api.GetErrorString;
  return api;
}

tn_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return TN_OK;
  return fail(TN_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace
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

// Rows of Θ(c) whose sorted left position is < pos: its rows are [row0, row0+R) for single-charge plans,
// and for MPO pair plans whole left pair segments l = (l1, l2), l − (c1, c2) ∈ [0, d−1]², in key order
static int64_t sector_rows_before(const tn_plan* p, int c, int64_t pos) {
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

tn_status tn_plan_slab_rows(const tn_plan* p, int c, int rank, int64_t* row_begin, int64_t* rows) {
  if (!p || !row_begin || !rows) return fail(TN_ERR_DIMENSION, "tn_plan_slab_rows: NULL");
  if (c < 0 || c >= p->nsec) return fail(TN_ERR_DOMAIN, "tn_plan_slab_rows: sector out of range");
  if (rank < 0 || rank >= p->world) return fail(TN_ERR_DOMAIN, "tn_plan_slab_rows: rank out of range");
  const int64_t b = sector_rows_before(p, c, p->bounds[rank]), e = sector_rows_before(p, c, p->bounds[rank + 1]);
  *row_begin = b;
  *rows = e - b;
  return TN_OK;
}

tn_status tn_theta_exec_sharded(const tn_plan* p, tn_stream stream, tn_comm* comm, double* gamma_k,
                                double* lambda_k, double* gamma_k1, double* lambda_l, double* lambda_r, double* U,
                                double* const* theta_out, int bcast_operands, int gather_mode) {
  if (!p || !comm) return fail(TN_ERR_DIMENSION, "tn_theta_exec_sharded: NULL plan/comm");
  if (p->world != comm->world || p->rank != comm->rank)
    return fail(TN_ERR_CONSISTENCY, "tn_theta_exec_sharded: plan world/rank differ from the communicator's");
  if (gather_mode != TN_GATHER_NONE && gather_mode != TN_GATHER_ROOT && gather_mode != TN_GATHER_SECTOR_OWNER)
    return fail(TN_ERR_DOMAIN, "tn_theta_exec_sharded: unknown gather_mode");
  if (!theta_out) return fail(TN_ERR_DIMENSION, "tn_theta_exec_sharded: NULL theta_out");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(TN_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded");
  cudaStream_t s = (cudaStream_t)stream;
  tn_status st;
  if (bcast_operands && p->world > 1) {
    st = nccl_check(api.GroupStart(), "ncclGroupStart");
    if (st != TN_OK) return st;
    const size_t n_gk = (size_t)(2 * p->chi[0] * p->chi[1]), n_gk1 = (size_t)(2 * p->chi[1] * p->chi[2]);
    ncclResult_t r = ncclSuccess;
    if (r == ncclSuccess) r = api.Broadcast(gamma_k, gamma_k, n_gk, ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(gamma_k1, gamma_k1, n_gk1, ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_k, lambda_k, (size_t)p->chi[1], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_l, lambda_l, (size_t)p->chi[0], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(lambda_r, lambda_r, (size_t)p->chi[2], ncclFloat64, 0, comm->comm, s);
    if (r == ncclSuccess) r = api.Broadcast(U, U, (size_t)(2 * p->u_size), ncclFloat64, 0, comm->comm, s);
    ncclResult_t r2 = api.GroupEnd();
    st = nccl_check(r != ncclSuccess ? r : r2, "operand broadcast");
    if (st != TN_OK) return st;
  }
  auto rows_before = [&](int c, int64_t pos) { return sector_rows_before(p, c, pos); };
  // Local slabs: where this rank receives a whole sector (ROOT: rank 0, SECTOR_OWNER: the sector's owner)
  // the caller passed the FULL Θ(c), so this rank's slab starts at row rows_before(c, r0).
  auto dest = [&](int c) { return gather_mode == TN_GATHER_ROOT ? 0 : p->owner[c]; };
  std::vector<double*> local(p->nsec, nullptr);
  for (int c = 0; c < p->nsec; ++c) {
    double* base = theta_out[c];
    if (gather_mode != TN_GATHER_NONE && p->world > 1 && dest(c) == p->rank && base)
      base += 2 * rows_before(c, p->r0) * p->C[c];
    local[c] = base;
  }
  st = tn_theta_exec(p, stream, gamma_k, lambda_k, gamma_k1, lambda_l, lambda_r, U, local.data());
  if (st != TN_OK || gather_mode == TN_GATHER_NONE || p->world == 1) return st;
  st = nccl_check(api.GroupStart(), "ncclGroupStart");
  if (st != TN_OK) return st;
  ncclResult_t r = ncclSuccess;
  for (int c = 0; c < p->nsec && r == ncclSuccess; ++c) {
    const int64_t C = p->C[c];
    const int to = dest(c);
    if (p->rank == to) {
      for (int src = 0; src < p->world && r == ncclSuccess; ++src) {
        if (src == to) continue;
        const int64_t s0 = rows_before(c, p->bounds[src]), s1 = rows_before(c, p->bounds[src + 1]);
        if (s1 > s0 && C > 0)
          r = api.Recv(theta_out[c] + 2 * s0 * C, (size_t)(2 * (s1 - s0) * C), ncclFloat64, src, comm->comm, s);
      }
    } else if (p->lR[c] * C > 0) {
      r = api.Send(theta_out[c], (size_t)(2 * p->lR[c] * C), ncclFloat64, to, comm->comm, s);
    }
  }
  ncclResult_t r2 = api.GroupEnd();
  return nccl_check(r != ncclSuccess ? r : r2, gather_mode == TN_GATHER_ROOT ? "Θ gather to root" : "Θ gather to sector owners");
}

}  // extern "C"
