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
#include "tn_internal.cuh"

namespace tn {

constexpr int MIX_THREADS = 128;
constexpr int MIX_WARPS = MIX_THREADS / 32;
constexpr int MIX_GROUPS_PER_TILE = 128;  // 8-groups per CTA tile (32 per warp)

__device__ __forceinline__ void dmma5(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Row stride (complex entries) of the staged Us: a quarter warp's B-fragment LDS.128 (two rows × 4
// consecutive u) then covers all 32 banks once.
__host__ __device__ __forceinline__ int us_stride(int UP) { return ((UP * 16) % 128 == 64) ? UP : UP + 4; }

struct SecRef {             // sector lo+u at the tile block's origin (row pl0, column pr0)
  const double2* base;      // (load table: nullptr for an empty center segment → P = 0)
  int64_t ld;
};

template <int KSM>
__device__ __forceinline__ void load_group(double2 (&a)[KSM], const SecRef* __restrict__ sec, int L, int64_t row,
                                           int col, bool valid, int q) {
#pragma unroll
  for (int ks = 0; ks < KSM; ++ks) {
    const int u = ks * 4 + q;
    a[ks] = make_double2(0.0, 0.0);
    if (valid && u < L) {
      const SecRef s = sec[u];
      if (s.base) a[ks] = __ldcs(s.base + row * s.ld + col);
    }
  }
}

template <int NT>  // NT = ⌈L/8⌉ output tiles of 8 sectors
__device__ __forceinline__ void mix_tile_warp(const MixTile& mt, const SecRef* __restrict__ sec,
                                              const SecRef* __restrict__ st_sec, const double2* __restrict__ Us,
                                              const double* __restrict__ UsS,
                                              int ust, int L, const int32_t* __restrict__ perm_l,
                                              const int32_t* __restrict__ perm_r, const double* __restrict__ ll,
                                              const double* __restrict__ lr, int warp, int lane) {
  constexpr int KSM = 2 * NT;
  const int g = lane >> 2, q = lane & 3;
  const int KS = (L + 3) >> 2;
  int k = warp;
  if (k >= mt.ne) return;
  auto coords = [&](int kk, int64_t& row, int& col) {
    const int grp = mt.e0 + kk;
    row = grp / mt.ngr;
    col = (int)(grp - row * mt.ngr) * 8 + g;
  };
  int64_t row;
  int col;
  coords(k, row, col);
  bool valid = col < mt.nr;
  double2 a[KSM];
  load_group<KSM>(a, sec, L, row, col, valid, q);
  while (true) {
    // prefetch the next group of this warp before computing the current one
    const int kn = k + MIX_WARPS;
    const bool has_next = kn < mt.ne;
    int64_t rown = 0;
    int coln = 0;
    bool validn = false;
    double2 an[KSM];
    if (has_next) {
      coords(kn, rown, coln);
      validn = coln < mt.nr;
      load_group<KSM>(an, sec, L, rown, coln, validn, q);
    }
    // Gauss 3-product form: T1 = Pr·Ur, T2 = Pi·Ui, T3 = (Pr+Pi)·(Ur+Ui); Re = T1−T2, Im = T3−T1−T2
    double acc[NT][6];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int x = 0; x < 6; ++x) acc[j][x] = 0.0;
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) {
      if (ks < KS) {
        const double as = a[ks].x + a[ks].y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int idx = (j * 8 + g) * ust + ks * 4 + q;  // B frag: Usᵀ[u = 4ks+q][t = 8j+g]
          const double2 b = Us[idx];
          const double bs = UsS[idx];
          dmma5(acc[j][0], acc[j][1], a[ks].x, b.x);  // T1
          dmma5(acc[j][2], acc[j][3], a[ks].y, b.y);  // T2
          dmma5(acc[j][4], acc[j][5], as, bs);        // T3
        }
      }
    }
    if (valid) {
      const double scale = ll[perm_l[mt.pl0 + row]] * lr[perm_r[mt.pr0 + col]];
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = j * 8 + 2 * q + h;
          if (t < L) {
            const SecRef s = st_sec[t];  // output sector lo+t (every output sector is stored)
            const double re = acc[j][h] - acc[j][2 + h];
            const double im = acc[j][4 + h] - acc[j][h] - acc[j][2 + h];
            __stcs(const_cast<double2*>(s.base) + row * s.ld + col, make_double2(re * scale, im * scale));
          }
        }
    }
    if (!has_next) break;
    k = kn;
    row = rown;
    col = coln;
    valid = validn;
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) a[ks] = an[ks];
  }
}

template <int NTMAX>
__global__ void __launch_bounds__(MIX_THREADS, (NTMAX <= 4 ? 4 : 2))
    k5_mix(const SectorParams sp, const MixTile* __restrict__ tiles, const int32_t* __restrict__ perm_l,
           const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
           const double2* __restrict__ U, int us_elems) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const MixTile mt = tiles[blockIdx.x];
  const int d = sp.d;
  const int c_l = mt.cl, c_r = mt.cr, n = c_l - c_r;
  const int lo = max(c_r, c_l - d + 1), hi = min(c_l, c_r + d - 1);
  const int L = hi - lo + 1;
  const int nlo = max(0, n - d + 1);
  const int sn = min(n, d - 1) - nlo + 1;
  const int TP = (L + 7) & ~7, UP = (L + 3) & ~3;
  const int ust = us_stride(UP);
  SecRef* ld_sec = reinterpret_cast<SecRef*>(smem_raw);           // load table (null if empty segment)
  SecRef* st_sec = ld_sec + 8 * NTMAX;                            // store table
  double2* Us = reinterpret_cast<double2*>(st_sec + 8 * NTMAX);   // U sub-block
  double* UsS = reinterpret_cast<double*>(Us + us_elems);          // Re + Im of every Us entry
  for (int u = threadIdx.x; u < L; u += MIX_THREADS) {
    const int cc = lo + u;
    const double2* base =
        sp.out[cc] + ((int64_t)mt.pl0 - sp.lrow0[cc]) * sp.ld[cc] + ((int64_t)mt.pr0 - sp.col0[cc]);
    const bool ne = (sp.cc_mask[cc >> 5] >> (cc & 31)) & 1u;
    ld_sec[u] = SecRef{ne ? base : nullptr, (int64_t)sp.ld[cc]};
    st_sec[u] = SecRef{base, (int64_t)sp.ld[cc]};
  }
  // Us[t][u] = U_n[i = c_l − (lo+t)][j = c_l − (lo+u)], zero-padded to TP × UP
  const double2* Ub = U + sp.ustart[n];
  for (int x = threadIdx.x; x < TP * UP; x += MIX_THREADS) {
    const int t = x / UP, u = x - t * UP;
    double2 v = make_double2(0.0, 0.0);
    if (t < L && u < L) v = __ldg(Ub + (c_l - lo - t - nlo) * sn + (c_l - lo - u - nlo));
    Us[t * ust + u] = v;
    UsS[t * ust + u] = v.x + v.y;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  switch (TP >> 3) {
#define TN_MIX_CASE(m)                                                                              \
  case m:                                                                                           \
    if constexpr (m <= NTMAX)                                                                       \
      mix_tile_warp<m>(mt, ld_sec, st_sec, Us, UsS, ust, L, perm_l, perm_r, ll, lr, warp, lane);   \
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
void build_mix_tiles(const tn_plan* p, std::vector<MixTile>& out) {
  out.clear();
  const auto& ol = p->off[0];
  const auto& orr = p->off[2];
  constexpr int BAND = 4;
  for (int cl = 0; cl <= p->N; ++cl) {
    const int64_t a0 = std::max<int64_t>(ol[cl], p->r0), a1 = std::min<int64_t>(ol[cl + 1], p->r1);
    for (int64_t band = a0; band < a1; band += BAND) {
      const int64_t rows = std::min<int64_t>(BAND, a1 - band);
      for (int cr = std::max(0, cl - 2 * p->d + 2); cr <= cl; ++cr) {
        const int64_t nr = orr[cr + 1] - orr[cr];
        if (nr == 0) continue;
        const int64_t ngr = (nr + 7) / 8;
        const int64_t G = rows * ngr;
        for (int64_t e0 = 0; e0 < G; e0 += MIX_GROUPS_PER_TILE) {
          MixTile t;
          t.cl = cl;
          t.cr = cr;
          t.e0 = (int32_t)e0;
          t.ne = (int32_t)std::min<int64_t>(MIX_GROUPS_PER_TILE, G - e0);
          t.nr = (int32_t)nr;
          t.ngr = (int32_t)ngr;
          t.pl0 = (int32_t)band;
          t.pr0 = (int32_t)orr[cr];
          out.push_back(t);
        }
      }
    }
  }
}

cudaError_t launch_mix(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                       const double2* U, cudaStream_t s) {
  if (p->nmix == 0) return cudaSuccess;
  const unsigned grid = (unsigned)p->nmix;
  const int L = p->max_mix;
  const int NT = (L + 7) >> 3;
  int smax = 0;  // largest staged Us over every L ≤ max_mix
  for (int l = 1; l <= L; ++l) {
    const int tp = (l + 7) & ~7, up = (l + 3) & ~3;
    smax = std::max(smax, tp * us_stride(up));
  }
#define TN_MIX_LAUNCH(M)                                                                                       \
  do {                                                                                                         \
    const size_t smem = (size_t)smax * (sizeof(double2) + sizeof(double)) + 2 * 8 * (M) * sizeof(SecRef);     \
    if (smem > 48 * 1024) {                                                                                    \
      cudaError_t e = cudaFuncSetAttribute(k5_mix<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
      if (e != cudaSuccess) return e;                                                                          \
    }                                                                                                          \
    k5_mix<M><<<grid, MIX_THREADS, smem, s>>>(sp, p->d_mix, p->d_perm[0], p->d_perm[2], ll, lr, U, smax);      \
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
}

}  // namespace tn
