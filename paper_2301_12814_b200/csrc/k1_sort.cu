// K1 — bond re-indexing: stable ascending counting sort of one bond by charge.
//
// PAPER.md:92 "we propose to sort the bonds according to their charges before GPU computation";
// PAPER.md:94 "bond indices are sorted such that c_{α_k} only increases as the bond index
// increases". Tie-break is stable (R1). One CTA per bond: histogram →
// exclusive scan → chunked stable scatter (warp match_any ranks within a chunk). Latency-bound
// (µs); it runs once per plan, off the hot path, on the plan's own stream — its CTAs are sized to fit
// next to the previous gate's K4/K5 so planning overlaps execution.
#include "tn_internal.cuh"

namespace tn {

constexpr int SORT_THREADS = 256;   // small enough to co-reside with a running K4/K5 (next gate's plan)
constexpr int SORT_WARPS = SORT_THREADS / 32;

__global__ void __launch_bounds__(SORT_THREADS) k1_sort_bonds(const SortArgs args, int N) {
  const int bond = blockIdx.x;
  const int32_t* __restrict__ q = args.q[bond];
  const int32_t* __restrict__ q2 = args.q2[bond];  // MPO pair plans: sort by the lexicographic key
  const int64_t chi = args.chi[bond];
  int32_t* __restrict__ perm = args.perm[bond];
  int32_t* __restrict__ qs = args.qs[bond];
  int32_t* __restrict__ off = args.off[bond];
  int32_t* __restrict__ err = args.err + bond;
  const int nq = q2 ? (N + 1) * (N + 1) : N + 1;   // number of (pair) charge keys ≤ MAX_SEC
  // dynamic shared memory sized by the key count: hist[nq+1], base[nq+1], wcnt[SORT_WARPS][nq]
  extern __shared__ int32_t k1_smem[];
  int32_t* hist = k1_smem;
  int32_t* base = hist + nq + 1;
  int32_t* wcnt_flat = base + nq + 1;
  auto wcnt = [&](int w, int v) -> int32_t& { return wcnt_flat[w * nq + v]; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i <= nq; i += SORT_THREADS) hist[i] = 0;
  __syncthreads();
  int bad = 0;
  auto key = [&](int64_t i) -> int {  // −1 for a charge outside [0, N]
    const int a = q[i];
    if (a < 0 || a > N) return -1;
    if (!q2) return a;
    const int b = q2[i];
    return (b < 0 || b > N) ? -1 : a * (N + 1) + b;
  };
  for (int64_t i = tid; i < chi; i += SORT_THREADS) {
    const int v = key(i);
    if (v < 0) {
      bad = 1;
      continue;
    }
    atomicAdd(&hist[v], 1);
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) *err = 1;
    return;
  }
  if (tid == 0) {
    int acc = 0;
    for (int v = 0; v < nq; ++v) {
      base[v] = acc;
      off[v] = acc;
      acc += hist[v];
    }
    off[nq] = acc;
  }
  __syncthreads();
  // Chunked stable scatter: a chunk of SORT_THREADS consecutive bonds at a time, in order.
  for (int64_t c0 = 0; c0 < chi; c0 += SORT_THREADS) {
    for (int i = tid; i < SORT_WARPS * nq; i += SORT_THREADS) wcnt_flat[i] = 0;
    __syncthreads();
    const int64_t i = c0 + tid;
    const bool valid = i < chi;
    const int v = valid ? key(i) : -1;
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    unsigned peers = __match_any_sync(0xffffffffu, v);
    peers &= active;
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank_in_warp == 0) wcnt(warp, v) = __popc(peers);
    __syncthreads();
    if (valid) {
      int pos = base[v] + rank_in_warp;
      for (int w = 0; w < warp; ++w) pos += wcnt(w, v);
      perm[pos] = (int32_t)i;
      qs[pos] = v;
    }
    __syncthreads();
    for (int v2 = tid; v2 < nq; v2 += SORT_THREADS) {
      int s = 0;
      for (int w = 0; w < SORT_WARPS; ++w) s += wcnt(w, v2);
      base[v2] += s;
    }
    __syncthreads();
  }
}

cudaError_t launch_sort_bonds(const SortArgs& a, int N, cudaStream_t s) {
  const int nq = a.q2[0] ? (N + 1) * (N + 1) : N + 1;
  const size_t smem = (size_t)(2 * (nq + 1) + SORT_WARPS * nq) * sizeof(int32_t);   // ≤ 41 KB at MAX_SEC keys
  k1_sort_bonds<<<3, SORT_THREADS, smem, s>>>(a, N);
  return cudaGetLastError();
}

}  // namespace tn
