// K5 — U-weighted scatter of the per-center-charge products into the N+1 Θ(c) sectors, with the
// outer λ^{[k−1]}·λ^{[k+1]} scaling fused (BASELINE.json north_star item (4); Eq. S5).
//
// For an element (α, β) with charges c_l, c_r, n = c_l − c_r, the four δ's of Eq. S5 leave
//   Θ(c)[α,β] = λl[α] λr[β] Σ_{c_c} U_n[c_l−c][c_l−c_c] · P_{c_c}[α,β],
//   c, c_c ∈ [lo, hi] = [max(c_r, c_l−d+1), min(c_l, c_r+d−1)]   (the SAME index set)
// i.e. the (L = hi−lo+1)-vector of P values at (α,β) is multiplied by a sub-block of U_n. K4 wrote
// P_{c_c} into the Θ(c_c) buffers, so each thread reads its whole vector into registers, mixes, and
// overwrites it in place: every Θ element is read once and written once (HBM-bound; 16 B loads and
// stores, consecutive lanes on consecutive β of one row → coalesced). P_{c_c} with an empty center
// segment is zero and never read (its buffer holds no P). Vector lengths are bucketed per warp into
// compile-time register arrays of 4·m entries.
#include "tn_internal.cuh"

namespace tn {

constexpr int MIX_THREADS = 128;

template <int ML>
__device__ __forceinline__ void mix_vec(const SectorParams& sp, int64_t pl, int64_t pr, int c_l, int c_r,
                                        int L, int Lw, double scale, const double2* __restrict__ U) {
  const int d = sp.d;
  const int lo = max(c_r, c_l - d + 1);
  double2 P[ML];
#pragma unroll
  for (int u = 0; u < ML; ++u) {
    P[u] = make_double2(0.0, 0.0);
    const int cc = lo + u;
    if (u < L && ((sp.cc_mask[cc >> 5] >> (cc & 31)) & 1u)) {
      const double2* src = sp.out[cc] + (pl - sp.lrow0[cc]) * sp.ld[cc] + (pr - sp.col0[cc]);
      P[u] = __ldcs(src);
    }
  }
  const int n = c_l - c_r;
  const int nlo = max(0, n - d + 1);
  const int sn = min(n, d - 1) - nlo + 1;
  // U_n[i][j], i = c_l − c, j = c_l − c_c = c_l − lo − u
  const double2* Ub = U + sp.ustart[n] + (c_l - lo - nlo);
  for (int t = 0; t < Lw; ++t) {
    if (t < L) {
      const int c = lo + t;
      const double2* urow = Ub + (c_l - c - nlo) * sn;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int u = 0; u < ML; ++u) {
        if (u < L) {
          const double2 w = __ldg(urow - u);
          re = fma(w.x, P[u].x, re);
          re = fma(-w.y, P[u].y, re);
          im = fma(w.x, P[u].y, im);
          im = fma(w.y, P[u].x, im);
        }
      }
      double2* dst = sp.out[c] + (pl - sp.lrow0[c]) * sp.ld[c] + (pr - sp.col0[c]);
      __stcs(dst, make_double2(re * scale, im * scale));
    }
  }
}

// MLMAX bounds the register arrays instantiated in this kernel (one instance per size class, so
// small-d problems do not pay the register footprint of the largest vector length).
template <int MLMAX>
__global__ void __launch_bounds__(MIX_THREADS) k5_mix(const SectorParams sp, const int32_t* __restrict__ qs_l,
                                                      const int32_t* __restrict__ qs_r,
                                                      const int32_t* __restrict__ perm_l,
                                                      const int32_t* __restrict__ perm_r,
                                                      const double* __restrict__ ll, const double* __restrict__ lr,
                                                      const double2* __restrict__ U, const int32_t* __restrict__ offr,
                                                      int64_t r0) {
  const int64_t pl = r0 + blockIdx.x;
  const int c_l = qs_l[pl];
  const int d = sp.d, N = sp.N;
  const int64_t b0 = offr[max(0, c_l - 2 * d + 2)];
  const int64_t b1 = offr[min(N, c_l) + 1];
  const int64_t pr = b0 + (int64_t)blockIdx.y * MIX_THREADS + threadIdx.x;
  if (b0 + (int64_t)blockIdx.y * MIX_THREADS >= b1) return;  // whole block past the row's columns
  const bool active = pr < b1;
  int c_r = 0, L = 0;
  if (active) {
    c_r = qs_r[pr];
    L = min(c_l, c_r + d - 1) - max(c_r, c_l - d + 1) + 1;
  }
  const int Lw = __reduce_max_sync(0xffffffffu, L);
  if (!active) return;
  const double scale = ll[perm_l[pl]] * lr[perm_r[pr]];
  switch ((Lw + 3) >> 2) {
#define TN_MIX_CASE(m)                                                  \
  case m:                                                               \
    if constexpr (4 * m <= MLMAX) mix_vec<4 * m>(sp, pl, pr, c_l, c_r, L, Lw, scale, U); \
    break;
    TN_MIX_CASE(1) TN_MIX_CASE(2) TN_MIX_CASE(3) TN_MIX_CASE(4)
    TN_MIX_CASE(5) TN_MIX_CASE(6) TN_MIX_CASE(7) TN_MIX_CASE(8)
    TN_MIX_CASE(9) TN_MIX_CASE(10) TN_MIX_CASE(11) TN_MIX_CASE(12)
    TN_MIX_CASE(13) TN_MIX_CASE(14) TN_MIX_CASE(15) TN_MIX_CASE(16)
#undef TN_MIX_CASE
    default:
      break;
  }
}

cudaError_t launch_mix(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                       const double2* U, cudaStream_t s, const int32_t* d_offr) {
  const int64_t rows = p->r1 - p->r0;
  if (rows <= 0) return cudaSuccess;
  // widest column range of any row: n = c_l − c_r ∈ [0, 2d−2]
  int64_t wmax = 0;
  const auto& offr = p->off[2];
  for (int cl = 0; cl <= p->N; ++cl) {
    int64_t w = offr[std::min(p->N, cl) + 1] - offr[std::max(0, cl - 2 * p->d + 2)];
    wmax = std::max(wmax, w);
  }
  if (wmax == 0) return cudaSuccess;
  dim3 grid((unsigned)rows, (unsigned)((wmax + MIX_THREADS - 1) / MIX_THREADS));
#define TN_MIX_LAUNCH(M)                                                                                 \
  k5_mix<M><<<grid, MIX_THREADS, 0, s>>>(sp, p->d_qs[0], p->d_qs[2], p->d_perm[0], p->d_perm[2], ll, lr, U, \
                                         d_offr, p->r0)
  if (p->max_mix <= 8)
    TN_MIX_LAUNCH(8);
  else if (p->max_mix <= 16)
    TN_MIX_LAUNCH(16);
  else if (p->max_mix <= 32)
    TN_MIX_LAUNCH(32);
  else if (p->max_mix <= 48)
    TN_MIX_LAUNCH(48);
  else
    TN_MIX_LAUNCH(64);
#undef TN_MIX_LAUNCH
  return cudaGetLastError();
}

}  // namespace tn
