// K45 — K4 contraction and K5 U-mix in ONE persistent kernel (DESIGN.md §4 "K45"): the mix of a row
// band runs on dedicated mixer warps while the contraction warps of every SM are already working on
// later bands, so K5's HBM-pattern-bound traffic overlaps the FP64 tensor-bound K4 instead of
// following it (two kernels: 2.55 + 0.78 ms at config 3).
//
// Same arithmetic as the two kernels (Eq. S5 with the product-once reformulation):
//   P_{c_c} = A_{c_c}·B_{c_c}   (consumer warps 0–7, producer warp 8: exactly k4_contract's tile loop)
//   Θ(c) = λlλr Σ_{c_c} U_n[c_l−c][c_l−c_c] P_{c_c}   (mixer warps 9–11: k5_mix's per-tile warp loop)
//
// Ordering. Rows of this rank's shard are cut into bands of K45_BAND sorted left positions. The plan
// lists K4 tiles band-major (by the first band a tile touches, heavy-first inside a band) and mix
// tiles band by band; need[b] = number of K4 tiles touching band b. A consumer CTA that finishes a
// tile makes its P stores visible (per-thread __threadfence, consumer named barrier) and adds 1 to
// done[b] for every band the tile touches. A mixer group waits (acquire load) until done[b] == need[b]
// before staging U and reading P of band b through L2 (ld.global.cg). Every CTA is resident (grid =
// SM count, one CTA per SM), and consumers never wait on mixers, so the waits cannot deadlock.
// In place, as in K5: a mixer lane reads all L values P_{c_c}[α,β] and writes all L values Θ(c)[α,β].
#include <cstdlib>

#include "k4_device.cuh"
#include "k5_mix.cuh"

namespace tn {

constexpr int K45_MIX_WARPS = 3;
constexpr int K45_THREADS = (K4_CONSUMER_WARPS + 1 + K45_MIX_WARPS) * 32;  // 12 warps: ≤ 168 registers

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int STAGES, int NTMAX>
__global__ void __launch_bounds__(K45_THREADS, 1)
    k45_fused(const GroupDesc* __restrict__ groups, const TileDesc* __restrict__ tiles, int ntiles,
              const double2* __restrict__ ap, const double2* __restrict__ bp, const SectorParams sp,
              const MixTile* __restrict__ mtiles, int nmix, const int32_t* __restrict__ perm_l,
              const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
              const double2* __restrict__ U, int us_elems, const int32_t* __restrict__ need,
              int32_t* __restrict__ done, int64_t r0, int dbg) {
  extern __shared__ __align__(128) uint8_t smem[];
  double2* sA = reinterpret_cast<double2*>(smem);
  double2* sB = sA + STAGES * CHUNK;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  SecRef* ld_sec = reinterpret_cast<SecRef*>(empty + STAGES);
  SecRef* st_sec = ld_sec + 8 * NTMAX;
  double2* Us = reinterpret_cast<double2*>(st_sec + 8 * NTMAX);
  double* UsS = reinterpret_cast<double*>(Us + us_elems);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], K4_CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp > K4_CONSUMER_WARPS) {
    // ---------------- mixers: warps 9..11, band by band ----------------
    const int mw = warp - K4_CONSUMER_WARPS - 1, mtid = tid - (K4_CONSUMER_WARPS + 1) * 32;
    constexpr int MIX_THR = K45_MIX_WARPS * 32;
    for (int m = (dbg & 1) ? nmix : blockIdx.x; m < nmix; m += gridDim.x) {  // dbg 1: no mix (timing study)
      const MixTile mt = mtiles[m];
      if (mtid == 0) {
        const int b = (int)((mt.pl0 - r0) / K45_BAND);
        const int want = need[b];
        while (ld_acquire(done + b) < want) __nanosleep(256);
      }
      asm volatile("bar.sync 2, %0;" ::"n"(MIX_THR) : "memory");  // band ready; previous tile finished
      int L, ust;
      mix_stage(mt, sp, U, ld_sec, st_sec, Us, UsS, mtid, MIX_THR, L, ust);
      asm volatile("bar.sync 2, %0;" ::"n"(MIX_THR) : "memory");
      switch (((L + 7) & ~7) >> 3) {
#define TN_MIX_CASE(q)                                                                                      \
  case q:                                                                                                   \
    if constexpr (q <= NTMAX)                                                                               \
      mix_tile_warp<q, K45_MIX_WARPS, true>(mt, ld_sec, st_sec, Us, UsS, ust, L, perm_l, perm_r, ll, lr, mw, \
                                            lane);                                                          \
    break;
        TN_MIX_CASE(1) TN_MIX_CASE(2) TN_MIX_CASE(3) TN_MIX_CASE(4)
        TN_MIX_CASE(5) TN_MIX_CASE(6) TN_MIX_CASE(7) TN_MIX_CASE(8)
#undef TN_MIX_CASE
        default:
          break;
      }
    }
    return;
  }

  if (warp == K4_CONSUMER_WARPS) {
    // ---------------- producer: one elected lane streams A/B chunks ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileDesc td = tiles[t];
        const GroupDesc g = groups[td.g];
        const double2* a = ap + g.a_off + (int64_t)td.mt * BM * g.K4;
        const double2* b = bp + g.b_off + (int64_t)td.nt * BN * g.K4;
        for (int kc = 0; kc * BK < g.K4; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t kcnt = (uint32_t)min(BK, g.K4 - kc * BK);
          const uint32_t bytes = kcnt * BM * (uint32_t)sizeof(double2);
          mbar_expect_tx(&full[stage], 2 * bytes);
          bulk_g2s(sA + stage * CHUNK, a + (int64_t)kc * CHUNK, bytes, &full[stage]);
          bulk_g2s(sB + stage * CHUNK, b + (int64_t)kc * CHUNK, bytes, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: 2×4 warps, 32×16 complex outputs each (as k4_contract) ----------------
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  TileDesc td_next;
  GroupDesc g_next;
  if (blockIdx.x < ntiles) {
    td_next = tiles[blockIdx.x];
    g_next = groups[td_next.g];
  }
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const TileDesc td = td_next;
    const GroupDesc g = g_next;
    if (t + (int)gridDim.x < ntiles) {
      td_next = tiles[t + gridDim.x];
      g_next = groups[td_next.g];
    }
    double acc[4][2][6];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[mi][ni][q] = 0.0;

    for (int kc = 0; kc * BK < g.K4; ++kc) {
      mbar_wait(&full[stage], phase);
      const int nks = min(BK, g.K4 - kc * BK) >> 2;
      const double2* As = sA + stage * CHUNK + wm * 128 + lane;
      const double2* Bs = sB + stage * CHUNK + wn * 64 + lane;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        if (ks < nks) {
          double2 a[4], b[2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) a[mi] = As[ks * 256 + mi * 32];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) b[ni] = Bs[ks * 256 + ni * 32];
          double bsum[2];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) bsum[ni] = b[ni].x + b[ni].y;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const double asum = a[mi].x + a[mi].y;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              double* c = acc[mi][ni];
              dmma(c[0], c[1], a[mi].x, b[ni].x);  // T1 += Ar·Br
              dmma(c[2], c[3], a[mi].y, b[ni].y);  // T2 += Ai·Bi
              dmma(c[4], c[5], asum, bsum[ni]);    // T3 += (Ar+Ai)·(Br+Bi)
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    double2* out = sp.out[g.cc];
    const int ld = sp.ld[g.cc];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int row = td.mt * BM + wm * 32 + mi * 8 + gq;
      if (row >= g.R) continue;
      double2* orow = out + (int64_t)row * ld;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        const int col = td.nt * BN + wn * 16 + ni * 8 + 2 * tq;
        const double* c = acc[mi][ni];
        const double re0 = c[0] - c[2], re1 = c[1] - c[3];
        const double im0 = c[4] - c[0] - c[2], im1 = c[5] - c[1] - c[3];
        if (col < g.C) orow[col] = make_double2(re0, im0);
        if (col + 1 < g.C) orow[col + 1] = make_double2(re1, im1);
      }
    }
    // publish: this tile's P is complete for every band it touches
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(K4_CONSUMER_WARPS * 32) : "memory");
    if (tid == 0) {
      const int64_t a0 = g.row0 + (int64_t)td.mt * BM - r0;
      const int64_t a1 = min((int64_t)g.row0 + g.R, (int64_t)g.row0 + (int64_t)td.mt * BM + BM) - r0;
      for (int64_t b = a0 / K45_BAND; b <= (a1 - 1) / K45_BAND; ++b) atomicAdd(done + b, 1);
    }
  }
}

static int k45_debug() {
  static const int v = [] {
    const char* e = getenv("TN_K45_ABLATE");  // timing studies only: 1 = mixers idle (Θ incomplete)
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int STAGES, int NTMAX>
static cudaError_t launch45(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                            const double2* U, int us_elems, cudaStream_t s) {
  const size_t smem = (size_t)STAGES * CHUNK * sizeof(double2) * 2 + 2 * STAGES * sizeof(uint64_t) +
                      2 * 8 * NTMAX * sizeof(SecRef) + (size_t)us_elems * (sizeof(double2) + sizeof(double));
  cudaError_t e = cudaFuncSetAttribute(k45_fused<STAGES, NTMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p->d_band_done, 0, sizeof(int32_t) * p->nbands, s);
  if (e != cudaSuccess) return e;
  k45_fused<STAGES, NTMAX><<<(unsigned)p->sm_count, K45_THREADS, smem, s>>>(
      p->d_groups, p->d_tiles, (int)p->ntiles, p->d_apanel, p->d_bpanel, sp, p->d_mix, (int)p->nmix, p->d_perm[0],
      p->d_perm[2], ll, lr, U, us_elems, p->d_band_need, p->d_band_done, p->r0, k45_debug());
  return cudaGetLastError();
}

// shared memory of the fused kernel for a given ring depth and longest mix vector
size_t k45_smem_bytes(int stages, int max_mix) {
  const int ntmax = max_mix <= 8 ? 1 : max_mix <= 16 ? 2 : max_mix <= 32 ? 4 : max_mix <= 48 ? 6 : 8;
  return (size_t)stages * CHUNK * sizeof(double2) * 2 + 2 * stages * sizeof(uint64_t) + 2 * 8 * ntmax * sizeof(SecRef) +
         (size_t)mix_us_elems(max_mix) * (sizeof(double2) + sizeof(double));
}

cudaError_t launch_fused(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                         const double2* U, cudaStream_t s) {
  if (p->ntiles == 0 && p->nmix == 0) return cudaSuccess;
  const int L = p->max_mix;
  const int us = mix_us_elems(L);
  const bool deep = k45_smem_bytes(6, L) <= 227 * 1024;
#define TN_F(ST, NT) return launch45<ST, NT>(p, sp, ll, lr, U, us, s)
  if (L <= 8) { if (deep) TN_F(6, 1); TN_F(5, 1); }
  if (L <= 16) { if (deep) TN_F(6, 2); TN_F(5, 2); }
  if (L <= 32) { if (deep) TN_F(6, 4); TN_F(5, 4); }
  if (L <= 48) { if (deep) TN_F(6, 6); TN_F(5, 6); }
  if (deep) TN_F(6, 8);
  TN_F(4, 8);
#undef TN_F
}

}  // namespace tn
