// Device code of the U-mix (K5, k5_mix.cu) and of the pair-plan mix K5P (tn_pair.cu). See k5_mix.cu for
// the design.
#pragma once
#include "tn_internal.cuh"

namespace tn {

constexpr int MIX_GROUPS_PER_TILE = 128;  // 8-groups per mix tile

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

template <int KSM, bool L2ONLY>
__device__ __forceinline__ void load_group(double2 (&a)[KSM], const SecRef* __restrict__ sec, int L, int64_t row,
                                           int col, bool valid, int q) {
#pragma unroll
  for (int ks = 0; ks < KSM; ++ks) {
    const int u = ks * 4 + q;
    a[ks] = make_double2(0.0, 0.0);
    if (valid && u < L) {
      const SecRef s = sec[u];
      // ld.global.cg: P is read once, so it skips L1, but with the normal L2 policy — the streaming
      // (evict-first) hint measured 2% slower on K5 (0.691 vs 0.675 ms at config 3)
      if (s.base) a[ks] = __ldcg(s.base + row * s.ld + col);
    }
  }
}

// L2ONLY: P was written by other SMs during the same kernel → bypass L1 (ld.global.cg; every load is .cg now)
// PF: groups further ahead (beyond the one held in registers) whose P lines are prefetched into L2
// (PF = 2 measured slower at configs 3 and 4: 0.82 vs 0.78 ms, 6.57 vs 6.05 ms)
// MULTI: the tile spans `nsub` sub-tiles of mt.ne 8-groups each, sub-tile i using sector tables sec + i·sstride
// and st_sec + i·sstride (K5P: several values of the other charge species in one CTA)
template <int NT, int NW, bool L2ONLY = false, int PF = 0, bool MULTI = false>  // NT = ⌈L/8⌉ output tiles of 8 sectors; NW warps per tile
__device__ __forceinline__ void mix_tile_warp(const MixTile& mt, const SecRef* __restrict__ sec0,
                                              const SecRef* __restrict__ st_sec0, const double2* __restrict__ Us,
                                              const double* __restrict__ UsS,
                                              int ust, int L, const int32_t* __restrict__ perm_l,
                                              const int32_t* __restrict__ perm_r, const double* __restrict__ ll,
                                              const double* __restrict__ lr, int warp, int lane, int nsub = 1,
                                              int sstride = 0) {
  constexpr int KSM = 2 * NT;
  const int g = lane >> 2, q = lane & 3;
  const int KS = (L + 3) >> 2;
  const int ntot = MULTI ? mt.ne * nsub : mt.ne;
  int k = warp;
  if (k >= ntot) return;
  auto coords = [&](int kk, int64_t& row, int& col, int& sub) {
    if (MULTI) {
      sub = kk / mt.ne;
      kk -= sub * mt.ne;
    } else {
      sub = 0;
    }
    const int grp = mt.e0 + kk;
    row = grp / mt.ngr;
    col = (int)(grp - row * mt.ngr) * 8 + g;
  };
  int64_t row;
  int col, sub;
  coords(k, row, col, sub);
  bool valid = col < mt.nr;
  const SecRef* sec = sec0 + (MULTI ? sub * sstride : 0);
  const SecRef* st_sec = st_sec0 + (MULTI ? sub * sstride : 0);
  double2 a[KSM];
  load_group<KSM, L2ONLY>(a, sec, L, row, col, valid, q);
  while (true) {
    // prefetch the next group of this warp before computing the current one
    const int kn = k + NW;
    const bool has_next = kn < ntot;
    int64_t rown = 0;
    int coln = 0, subn = 0;
    bool validn = false;
    double2 an[KSM];
    if (has_next) {
      coords(kn, rown, coln, subn);
      validn = coln < mt.nr;
      load_group<KSM, L2ONLY>(an, MULTI ? sec0 + subn * sstride : sec, L, rown, coln, validn, q);
    }
    if (PF > 0 && k + (PF + 1) * NW < ntot) {  // L2 prefetch PF groups further ahead (no registers held)
      int64_t rp;
      int cp, sp_;
      coords(k + (PF + 1) * NW, rp, cp, sp_);
      if (cp < mt.nr)
#pragma unroll
        for (int ks = 0; ks < KSM; ++ks) {
          const int u = ks * 4 + q;
          if (u < L && sec[u].base)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(sec[u].base + rp * sec[u].ld + cp));
        }
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
      const double scale = ll ? ll[perm_l[mt.pl0 + row]] * lr[perm_r[mt.pr0 + col]] : 1.0;  // ll = nullptr: no λ
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = j * 8 + 2 * q + h;
          if (t < L) {
            const SecRef s = st_sec[t];  // output sector lo+t (every output sector is stored)
            const double re = acc[j][h] - acc[j][2 + h];
            const double im = acc[j][4 + h] - acc[j][h] - acc[j][2 + h];
            __stcg(const_cast<double2*>(s.base) + row * s.ld + col, make_double2(re * scale, im * scale));
          }
        }
    }
    if (!has_next) break;
    k = kn;
    row = rown;
    col = coln;
    valid = validn;
    if (MULTI) {
      sec = sec0 + subn * sstride;
      st_sec = st_sec0 + subn * sstride;
    }
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) a[ks] = an[ks];
  }
}

// Stage a mix tile's sector tables and U sub-block in shared memory (nthr threads, index tid).
// Layout: ld_sec[8·NTMAX], st_sec[8·NTMAX], Us[us_elems] (complex), UsS[us_elems] (Re+Im).
__device__ __forceinline__ void mix_stage(const MixTile& mt, const SectorParams& sp, const double2* __restrict__ U,
                                          SecRef* ld_sec, SecRef* st_sec, double2* Us, double* UsS, int tid, int nthr,
                                          int& L, int& ust) {
  const int d = sp.d;
  const int c_l = mt.cl, c_r = mt.cr, n = c_l - c_r;
  const int lo = max(c_r, c_l - d + 1), hi = min(c_l, c_r + d - 1);
  L = hi - lo + 1;
  const int nlo = max(0, n - d + 1);
  const int sn = min(n, d - 1) - nlo + 1;
  const int TP = (L + 7) & ~7, UP = (L + 3) & ~3;
  ust = us_stride(UP);
  for (int u = tid; u < L; u += nthr) {
    const int cc = lo + u;
    const SecEntry e = sp.sec[cc];
    const int64_t off = ((int64_t)mt.pl0 - e.lrow0) * e.ld + ((int64_t)mt.pr0 - e.col0);
    const double2* base = e.out + off;
    const bool ne = e.nonempty;
    // P is read in place from Θ(c_c), or from a local workspace when Θ goes elsewhere (tn_theta_exec_remote)
    const double2* lbase = e.src ? e.src + off : base;
    ld_sec[u] = SecRef{ne ? lbase : nullptr, (int64_t)e.ld};
    st_sec[u] = SecRef{base, (int64_t)e.ld};
  }
  // Us[t][u] = U_n[i = c_l − (lo+t)][j = c_l − (lo+u)], zero-padded to TP × UP
  const double2* Ub = U + sp.ustart[n];
  for (int x = tid; x < TP * UP; x += nthr) {
    const int t = x / UP, u = x - t * UP;
    double2 v = make_double2(0.0, 0.0);
    if (t < L && u < L) v = __ldg(Ub + (c_l - lo - t - nlo) * sn + (c_l - lo - u - nlo));
    Us[t * ust + u] = v;
    UsS[t * ust + u] = v.x + v.y;
  }
}

// largest staged Us (complex entries) over every L ≤ max_mix
inline int mix_us_elems(int max_mix) {
  int smax = 0;
  for (int l = 1; l <= max_mix; ++l) {
    const int tp = (l + 7) & ~7, up = (l + 3) & ~3;
    smax = std::max(smax, tp * us_stride(up));
  }
  return smax;
}

}  // namespace tn
