// K5 — U-weighted scatter of the per-center-charge products into the N+1 Θ(c) sectors, with the
// outer λ^{[k−1]}·λ^{[k+1]} scaling fused (BASELINE.json north_star item (4); Eq. S5).
//
// For an element (α, β) with charges c_l, c_r, n = c_l − c_r, the four δ's of Eq. S5 leave
//   Θ(c)[α,β] = λl[α] λr[β] Σ_{c_c} U_n[c_l−c][c_l−c_c] · P_{c_c}[α,β],
//   c, c_c ∈ [lo, hi] = [max(c_r, c_l−d+1), min(c_l, c_r+d−1)]   (the SAME index set)
// K4 wrote P_{c_c} into the Θ(c_c) buffers; K5 mixes every element's L = hi−lo+1 values in place
// (each Θ element read once and written once: HBM-bound, 2 × 16 B per element).
//
// B200 design (DESIGN.md §4 "K5"):
//  * Work unit = a tile of ≤ MIX_GROUPS_PER_TILE "8-groups" (8 consecutive columns of one row) of ONE
//    (c_l, c_r) charge block, so n, L and the U sub-block Us[t][u] = U_n[c_l−lo−t][c_l−lo−u] are uniform
//    per CTA (the charge-sorted layout of PAPER.md:92-94 makes the U lookup uniform). The CTA stages Us
//    (zero-padded, bank-conflict-free stride) and a per-sector base-pointer table in shared memory.
//  * Over a tile the mix is the small GEMM Θᵀ(E×L) = Pᵀ(E×L)·Usᵀ(L×L) on the FP64 tensor pipe
//    (DMMA.8x8x4): a warp takes one 8-group (M = 8), K = u in steps of 4, N = t in tiles of 8. A-fragment
//    lane (g, q) loads P_{lo+u}[column g] (8 lanes → 128 contiguous bytes per sector); C-fragment lane
//    (g, q) stores Θ(lo+t)[column g], t = 2q, 2q+1 — a lane owns one element, so λl·λr is a per-lane
//    scalar. Registers stay small (⌈L/4⌉ complex per lane per group + ⌈L/8⌉ accumulator tiles).
//  * Each warp prefetches its next group's A fragments before the MMAs of the current one.
//  * Tiles are one row × one c_r block, issued row-major: what decides the HBM rate here is the ORDER
//    in which concurrently running CTAs touch the sector rows (a pure copy runs at 5.2–5.4 TB/s when
//    one row α is swept across consecutive c_r blocks, 2.8–3.5 TB/s when tiles are block-major,
//    whatever the per-instruction shape: tools/probe_mix_bw.cu, profiles/r01_probe_mix_bw.jsonl).
//  * P_{c_c} of an empty center segment is zero and never read.
//  * Register classes: the warp loop's registers grow with ⌈L/8⌉, and one kernel sized for the largest L
//    (128 registers at L = 32) capped every tile at 16 warps per SM. Tiles are therefore issued as up to
//    four launches by L (≤ 8: 56 registers, 8 CTAs/SM; ≤ 16: 72, 7 CTAs/SM; ≤ 32: 128; larger), each
//    keeping the band-major order: config 3 0.78 → 0.72 ms, config 4 6.05 → 4.30 ms.
#include <cstdlib>

#include "k5_mix.cuh"

namespace tn {

constexpr int MIX_THREADS = 128;
constexpr int MIX_WARPS = MIX_THREADS / 32;
#ifndef K5_SMALL_MINB
#define K5_SMALL_MINB 7   // CTAs per SM for the L ≤ 16 instantiations (≤ 72 registers, no spills)
#endif

template <int NTMAX>
__global__ void __launch_bounds__(MIX_THREADS, (NTMAX == 1 ? 8 : NTMAX == 2 ? K5_SMALL_MINB : NTMAX <= 4 ? 4 : 2))
    k5_mix(const SectorParams sp, const MixTile* __restrict__ tiles, const int32_t* __restrict__ perm_l,
           const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
           const double2* __restrict__ U, int us_elems) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const MixTile mt = tiles[blockIdx.x];
  SecRef* ld_sec = reinterpret_cast<SecRef*>(smem_raw);           // load table (null if empty segment)
  SecRef* st_sec = ld_sec + 8 * NTMAX;                            // store table
  double2* Us = reinterpret_cast<double2*>(st_sec + 8 * NTMAX);   // U sub-block
  double* UsS = reinterpret_cast<double*>(Us + us_elems);          // Re + Im of every Us entry
  int L, ust;
  mix_stage(mt, sp, U, ld_sec, st_sec, Us, UsS, threadIdx.x, MIX_THREADS, L, ust);
  const int TP = (L + 7) & ~7;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  switch (TP >> 3) {
#define TN_MIX_CASE(m)                                                                              \
  case m:                                                                                           \
    if constexpr (m <= NTMAX)                                                                       \
      mix_tile_warp<m, MIX_WARPS>(mt, ld_sec, st_sec, Us, UsS, ust, L, perm_l, perm_r, ll, lr, warp, lane);   \
    break;
    TN_MIX_CASE(1) TN_MIX_CASE(2) TN_MIX_CASE(3) TN_MIX_CASE(4)
    TN_MIX_CASE(5) TN_MIX_CASE(6) TN_MIX_CASE(7) TN_MIX_CASE(8)
#undef TN_MIX_CASE
    default:
      break;
  }
}

// Host: a tile = a band of rows × one c_r block (≈ MIX_GROUPS_PER_TILE 8-groups, so the per-CTA U
// staging is amortised), tiles issued band-major (row band, then c_r): concurrently running CTAs cover
// the same rows across consecutive c_r blocks, i.e. the sector rows are swept contiguously
// (tools/probe_mix_bw.cu: 5.2–5.4 TB/s row-major vs 2.8–3.5 TB/s block-major for a pure copy).
void build_mix_tiles(tn_plan* p, std::vector<MixTile>& out) {
  // classes: L ≤ 8, ≤ 16, ≤ 32, > 32 (one launch per register class), each in band-major order. Two passes — count,
  // then write every tile straight into its class's range — keep this host loop (on the per-gate plan's path)
  // free of reallocations and concatenation copies.
  const auto& ol = p->off[0];
  const auto& orr = p->off[2];
  constexpr int BAND = 4;  // 2 / 8 / 16 measured: 0.714 / 0.763 / 0.779 ms at config 3, 4.34 / 4.31 / 4.28 at config 4
  const int d = p->d;
  auto cls = [d](int cl, int cr) {
    const int L = std::min(cl, cr + d - 1) - std::max(cr, cl - d + 1) + 1;
    return L <= 8 ? 0 : L <= 16 ? 1 : L <= 32 ? 2 : 3;
  };
  auto walk = [&](auto&& emit) {
    for (int cl = 0; cl <= p->N; ++cl) {
      const int64_t a0 = std::max<int64_t>(ol[cl], p->r0), a1 = std::min<int64_t>(ol[cl + 1], p->r1);
      for (int64_t band = a0, rows = 0; band < a1; band += rows) {
        rows = std::min<int64_t>(BAND, a1 - band);
        for (int cr = std::max(0, cl - 2 * d + 2); cr <= cl; ++cr) {
          const int64_t nr = orr[cr + 1] - orr[cr];
          if (nr == 0) continue;
          const int64_t ngr = (nr + 7) / 8, G = rows * ngr;
          for (int64_t e0 = 0; e0 < G; e0 += MIX_GROUPS_PER_TILE) emit(cl, cr, band, nr, ngr, G, e0);
        }
      }
    }
  };
  int64_t cnt[4] = {0, 0, 0, 0};
  walk([&](int cl, int cr, int64_t, int64_t, int64_t, int64_t, int64_t) { ++cnt[cls(cl, cr)]; });
  int64_t at[4] = {0, cnt[0], cnt[0] + cnt[1], cnt[0] + cnt[1] + cnt[2]};
  out.resize((size_t)(at[3] + cnt[3]));
  MixTile* o = out.data();
  walk([&](int cl, int cr, int64_t band, int64_t nr, int64_t ngr, int64_t G, int64_t e0) {
    MixTile& t = o[at[cls(cl, cr)]++];
    t.cl = cl;
    t.cr = cr;
    t.e0 = (int32_t)e0;
    t.ne = (int32_t)std::min<int64_t>(MIX_GROUPS_PER_TILE, G - e0);
    t.nr = (int32_t)nr;
    t.ngr = (int32_t)ngr;
    t.pl0 = (int32_t)band;
    t.pr0 = (int32_t)orr[cr];
  });
  p->nmix_cls[0] = cnt[0];
  p->nmix_cls[1] = cnt[1];
  p->nmix_cls[2] = cnt[2];
}

cudaError_t launch_mix(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                       const double2* U, cudaStream_t s, int first_class) {
  if (p->nmix == 0) return cudaSuccess;
  // one launch per register class: L ≤ 8 (56 registers → 8 CTAs per SM), L ≤ 16 (72 → 7), L ≤ 32 (128 → 4),
  // the rest (NT 6/8 instantiations)
  auto one = [&](const MixTile* tiles, int64_t n, int L, cudaStream_t s) -> cudaError_t {
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)n;
    const int NT = (L + 7) >> 3;
    const int smax = mix_us_elems(L);
#define TN_MIX_LAUNCH(M)                                                                                       \
  do {                                                                                                         \
    const size_t smem = (size_t)smax * (sizeof(double2) + sizeof(double)) + 2 * 8 * (M) * sizeof(SecRef);     \
    if (smem > 48 * 1024) {                                                                                    \
      cudaError_t e = cudaFuncSetAttribute(k5_mix<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
      if (e != cudaSuccess) return e;                                                                          \
    }                                                                                                          \
    k5_mix<M><<<grid, MIX_THREADS, smem, s>>>(sp, tiles, p->d_perm[0], p->d_perm[2], ll, lr, U, smax);         \
  } while (0)
    if (NT <= 1)
      TN_MIX_LAUNCH(1);
    else if (NT <= 2)
      TN_MIX_LAUNCH(2);
    else if (NT <= 4)
      TN_MIX_LAUNCH(4);
    else if (NT <= 6)
      TN_MIX_LAUNCH(6);
    else
      TN_MIX_LAUNCH(8);
#undef TN_MIX_LAUNCH
    return cudaGetLastError();
  };
  const int L = p->max_mix;
  const int64_t n0 = p->nmix_cls[0], n1 = p->nmix_cls[1], n2 = p->nmix_cls[2], n3 = p->nmix - n0 - n1 - n2;
  const MixTile* t[4] = {p->d_mix, p->d_mix + n0, p->d_mix + n0 + n1, p->d_mix + n0 + n1 + n2};
  const int64_t n[4] = {first_class <= 0 ? n0 : 0, first_class <= 1 ? n1 : 0, first_class <= 2 ? n2 : 0, n3};
  const int Lc[4] = {std::min(L, 8), std::min(L, 16), std::min(L, 32), L};
  static const bool concurrent = getenv("TN_K5_SERIAL") == nullptr;
  if (!concurrent) {
    for (int c = 0; c < 4; ++c) {
      cudaError_t e = one(t[c], n[c], Lc[c], s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // the classes touch disjoint elements: run them concurrently (their tails and occupancy overlap) on
  // per-thread auxiliary streams forked from and joined back into s
  AuxStreams* ap = nullptr;
  if (cudaError_t ea = aux_streams(s, &ap); ea != cudaSuccess) return ea;
  AuxStreams& aux = *ap;
  cudaError_t e = cudaEventRecord(aux.fork, s);
  for (int c = 1; c < 4 && e == cudaSuccess; ++c) {
    if (n[c] == 0) continue;
    e = cudaStreamWaitEvent(aux.st[c - 1], aux.fork, 0);
    if (e == cudaSuccess) e = one(t[c], n[c], Lc[c], aux.st[c - 1]);
    if (e == cudaSuccess) e = cudaEventRecord(aux.join[c - 1], aux.st[c - 1]);
  }
  if (e == cudaSuccess) e = one(t[0], n[0], Lc[0], s);
  for (int c = 1; c < 4 && e == cudaSuccess; ++c)
    if (n[c]) e = cudaStreamWaitEvent(s, aux.join[c - 1], 0);
  return e;
}

}  // namespace tn
