// K3O + K4O — the contraction P_{c_c} = A_{c_c} · B_{c_c} of K4 run as an FP64-accurate
// emulation on the tcgen05 INT8 tensor cores (Ozaki splitting; DESIGN.md §4 "K3O/K4O").
//
// Splitting (K3O). For a real operand X and a row i (A) or column j (B), e = ilogb(max|x|) + 1 so
// x·2^−e ∈ (−1, 1); the signed 7-bit slices s_1..s_S come from  x ← 128·x, s ← trunc(x), x ← x − s
// (every step exact in FP64), so x·2^−e = Σ_p s_p 2^−7p + r, |r| < 2^−7S. The real and imaginary parts
// of a complex row/column share one exponent (max over both), so the four real products of a complex
// product carry the same scale and can be summed in one int32 accumulator:
//   Re P = Σ_{p+q ≤ S+1} 2^{e_i+f_j−7(p+q)} (Ar_p Br_q + Ai_p·(−Bi)_q),  Im P = … (Ar_p Bi_q + Ai_p Br_q)
// Slices are written in the UMMA canonical K-major SWIZZLE_NONE layout (8-row × 16-byte core matrices,
// a 128×32 or 64×32 tile contiguous), grouped per (row tile, K step): [plane (Ar, Ai)][slice] for A and
// [plane (Br, −Bi, Bi, Br)][slice] for B, so one stage of K4O is ONE contiguous bulk copy per operand.
//
// Contraction (K4O). Persistent CTA per SM, 10 warps: warp 0 streams stages with cp.async.bulk (TMA);
// warp 1 owns TMEM (512 columns) and one elected thread issues tcgen05.mma.cta_group::1.kind::i8
// (M=128, N=64, K=32) into one int32 accumulator per diagonal m = p+q (S × 64 columns) — a tile is done
// in two passes (Re, Im) that stream the same A stages against different B planes; warps 2–9 drain
// TMEM with tcgen05.ld, recombine Σ_m 2^−7m D_m in FP64, apply 2^{e_i+f_j}, and store P.
// Every int32 accumulator is exact: |D_m| ≤ 2·(m−1)·K·127² < 2^31 for K ≤ 2048.
#include <cmath>
#include <cstdio>

#include "tn_internal.cuh"

namespace tn {

// byte offset of element (r, k) (k < 32) inside one canonical rows×32 K-major tile
__host__ __device__ __forceinline__ int oz_canon(int r, int k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

template <int S>
__device__ __forceinline__ void slice16(const double* x16, uint4 (&out)[S]) {
  // 16 values in (−1,1) → S uint4 of packed int8 slices
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = x16[i];
#pragma unroll
  for (int p = 0; p < S; ++p) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      x[i] *= 128.0;
      const double t = trunc(x[i]);
      x[i] -= t;
      w[i >> 2] |= ((uint32_t)(int32_t)t & 0xFFu) << (8 * (i & 3));
    }
    out[p] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---- K3O(A): one warp per (padded) row of a group --------------------------------------------
template <int S>
__global__ void __launch_bounds__(256) k3o_rows(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_l,
                                                const int32_t* __restrict__ perm_c, const double2* __restrict__ gk,
                                                int64_t ld_gk, const double* __restrict__ lk, int8_t* __restrict__ oa,
                                                int32_t* __restrict__ oea) {
  const OzGroup g = groups[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  if (r >= g.nmt * OZ_BM) return;
  const bool valid = r < g.R;
  const int64_t a = valid ? perm_l[g.row0 + r] : 0;
  const double2* grow = gk + a * ld_gk;
  double mx = 0.0;
  if (valid)
    for (int k = lane; k < g.K; k += 32) {
      const int32_t gc = perm_c[g.k0 + k];
      const double2 v = grow[gc];
      const double s = lk[gc];
      mx = fmax(mx, fmax(fabs(v.x * s), fabs(v.y * s)));
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = mx > 0.0 ? ilogb(mx) + 1 : 0;
  if (lane == 0 && valid) oea[g.ea_off + r] = e;
  const int mt = r / OZ_BM, rr = r % OZ_BM;
  for (int c = lane; c < g.Kp / 16; c += 32) {
    double re[16], im[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = c * 16 + i;
      re[i] = im[i] = 0.0;
      if (valid && k < g.K) {
        const int32_t gc = perm_c[g.k0 + k];
        const double2 v = grow[gc];
        const double s = lk[gc];
        re[i] = ldexp(v.x * s, -e);
        im[i] = ldexp(v.y * s, -e);
      }
    }
    const int kc = c >> 1;
    int8_t* base = oa + g.a_off + (int64_t)(mt * g.nkc + kc) * (2 * S) * OZ_A_TILE + oz_canon(rr, (c & 1) * 16);
    uint4 sl[S];
    slice16<S>(re, sl);
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(base + (int64_t)p * OZ_A_TILE) = sl[p];
    slice16<S>(im, sl);
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(base + (int64_t)(S + p) * OZ_A_TILE) = sl[p];
  }
}

// ---- K3O(B): lane = column, one warp per 32 (padded) columns of a group -------------------------
template <int S>
__global__ void __launch_bounds__(256) k3o_cols(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_c,
                                                const int32_t* __restrict__ perm_r, const double2* __restrict__ gk1,
                                                int64_t ld_gk1, int8_t* __restrict__ ob, int32_t* __restrict__ oeb) {
  const OzGroup g = groups[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (blockIdx.x * 8 + warp) * 32 + lane;
  if ((blockIdx.x * 8 + warp) * 32 >= g.nnt * OZ_BN) return;  // warp-uniform
  const bool valid = j < g.C;
  const int64_t pc = valid ? perm_r[g.col0 + j] : 0;
  double mx = 0.0;
  if (valid)
    for (int k = 0; k < g.K; ++k) {
      const double2 v = gk1[(int64_t)perm_c[g.k0 + k] * ld_gk1 + pc];
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
  const int e = mx > 0.0 ? ilogb(mx) + 1 : 0;
  if (valid) oeb[g.eb_off + j] = e;
  const int nt = j / OZ_BN, jj = j % OZ_BN;
  for (int c = 0; c < g.Kp / 16; ++c) {
    double re[16], im[16], nim[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = c * 16 + i;
      re[i] = im[i] = 0.0;
      if (valid && k < g.K) {
        const double2 v = gk1[(int64_t)perm_c[g.k0 + k] * ld_gk1 + pc];
        re[i] = ldexp(v.x, -e);
        im[i] = ldexp(v.y, -e);
      }
      nim[i] = -im[i];
    }
    const int kc = c >> 1;
    int8_t* base = ob + g.b_off + (int64_t)(nt * g.nkc + kc) * (4 * S) * OZ_B_TILE + oz_canon(jj, (c & 1) * 16);
    uint4 sl[S];
    slice16<S>(re, sl);  // planes 0 and 3: Br
#pragma unroll
    for (int p = 0; p < S; ++p) {
      *reinterpret_cast<uint4*>(base + (int64_t)p * OZ_B_TILE) = sl[p];
      *reinterpret_cast<uint4*>(base + (int64_t)(3 * S + p) * OZ_B_TILE) = sl[p];
    }
    slice16<S>(nim, sl);  // plane 1: −Bi
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(base + (int64_t)(S + p) * OZ_B_TILE) = sl[p];
    slice16<S>(im, sl);  // plane 2: Bi
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(base + (int64_t)(2 * S + p) * OZ_B_TILE) = sl[p];
  }
}

// ---- K4O ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ob_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void ob_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void ob_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void ob_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(s32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void ob_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   s32(dst)),
               "l"(src), "r"(bytes), "r"(s32(bar))
               : "memory");
}
// UMMA smem descriptor, K-major SWIZZLE_NONE: LBO = 128 B (K-adjacent core matrices), SBO = 256 B
// (next 8-row group of a 32-byte-wide tile); version 1 (sm_100)
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                              ((uint32_t)(OZ_BM >> 4) << 24);  // s8×s8→s32, K-major, M=128, N=64

constexpr int OZ_THREADS = 10 * 32;

// One ring stage = one "half step": A plane h (S slices, 128×32 each) and B plane 2·pass + h (S slices,
// 64×32 each) of one K step of one tile; the Re pass pairs (Ar, Br), (Ai, −Bi), the Im pass (Ar, Bi),
// (Ai, Br). Small stages let the ring run 5–6 deep (the v1 ring of whole K steps was only 2 deep).
template <int S>
__device__ __forceinline__ void oz_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile("{\n .reg .pred pp;\n setp.ne.b32 pp, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n" ::"r"(d),
               "l"(da), "l"(db), "r"(OZ_IDESC), "r"(acc));
}

template <int S, int OZ_STAGES>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k4o_contract(const OzGroup* __restrict__ groups, const OzTile* __restrict__ tiles, int ntiles,
                 const int8_t* __restrict__ oa, const int8_t* __restrict__ ob, const int32_t* __restrict__ oea,
                 const int32_t* __restrict__ oeb, const SectorParams sp) {
  constexpr int A_HS = S * OZ_A_TILE, B_HS = S * OZ_B_TILE;   // one plane of one K step
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + OZ_STAGES * A_HS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + OZ_STAGES * B_HS);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* acc_full = empty + OZ_STAGES;
  uint64_t* acc_empty = acc_full + 1;  // one per diagonal m = 2..S+1 (index m − 2)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      ob_init(&full[s], 1);
      ob_init(&empty[s], 1);
    }
    ob_init(acc_full, 1);
    for (int m = 0; m < S; ++m) ob_init(&acc_empty[m], 8);  // the 8 epilogue warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const OzTile td = tiles[t];
        const OzGroup g = groups[td.g];
        const int8_t* a_t = oa + g.a_off + (int64_t)td.mt * g.nkc * 2 * A_HS;
        const int8_t* b_t = ob + g.b_off + (int64_t)td.nt * g.nkc * 4 * B_HS;
        for (int pass = 0; pass < 2; ++pass)
          for (int kc = 0; kc < g.nkc; ++kc)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              ob_wait(&empty[stage], phase ^ 1);
              ob_expect_tx(&full[stage], A_HS + B_HS);
              ob_bulk(sA + stage * A_HS, a_t + (int64_t)(kc * 2 + h) * A_HS, A_HS, &full[stage]);
              ob_bulk(sB + stage * B_HS, b_t + (int64_t)(kc * 4 + pass * 2 + h) * B_HS, B_HS, &full[stage]);
              if (++stage == OZ_STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int nkc = groups[tiles[t].g].nkc;
        for (int pass = 0; pass < 2; ++pass) {
          for (int kc = 0; kc < nkc; ++kc) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              ob_wait(&full[stage], phase);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              // descriptor of slice p = base + p·tile bytes (16-byte units; no carry out of the 14-bit field)
              const uint64_t da = oz_desc(s32(sA + stage * A_HS)), db = oz_desc(s32(sB + stage * B_HS));
              if (kc == 0 && h == 0) {
                // first half step of a pass: diagonal by diagonal, each once the epilogue has drained it
#pragma unroll
                for (int m = 2; m <= S + 1; ++m) {
                  ob_wait(&acc_empty[m - 2], acc_phase ^ 1);
                  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                  for (int p = 1; p <= S; ++p) {
                    const int q = m - p;
                    if (q < 1 || q > S) continue;
                    oz_mma<S>(tmem + (uint32_t)(m - 2) * OZ_BN, da + (uint64_t)((p - 1) * OZ_A_TILE >> 4),
                              db + (uint64_t)((q - 1) * OZ_B_TILE >> 4), p == (m - S > 1 ? m - S : 1) ? 0u : 1u);
                  }
                }
              } else {
#pragma unroll
                for (int p = 1; p <= S; ++p)
#pragma unroll
                  for (int q = 1; q <= S + 1 - p; ++q)
                    oz_mma<S>(tmem + (uint32_t)(p + q - 2) * OZ_BN, da + (uint64_t)((p - 1) * OZ_A_TILE >> 4),
                              db + (uint64_t)((q - 1) * OZ_B_TILE >> 4), 1u);
              }
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               s32(&empty[stage]))
                           : "memory");
              if (++stage == OZ_STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           s32(acc_full))
                       : "memory");
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..9 ----------------
    const int quad = warp & 3;              // TMEM lanes 32·quad .. +31 (a warp's accessible quadrant)
    const int half = (warp - 2) >> 2;       // columns 32·half .. +31
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const OzTile td = tiles[t];
      const OzGroup g = groups[td.g];
      const int row = td.mt * OZ_BM + quad * 32 + lane;
      const int col0 = td.nt * OZ_BN + half * 32;
      // exponents first (global loads off the accumulator critical path)
      const int er = row < g.R ? oea[g.ea_off + row] : 0;
      // lane j holds the exponent of column col0 + j (broadcast with shuffles below)
      const int ec_lane = (col0 + lane < g.C) ? oeb[g.eb_off + col0 + lane] : 0;
      double re[32];
      for (int pass = 0; pass < 2; ++pass) {
        ob_wait(acc_full, acc_phase);
        acc_phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        double v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0;
#pragma unroll 1
        for (int m = 2; m <= S + 1; ++m) {
          const double w = ldexp(1.0, -7 * m);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t r[16];
            const uint32_t ta =
                tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(m - 2) * OZ_BN + half * 32 + hh * 16;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) v[hh * 16 + j] = fma((double)(int32_t)r[j], w, v[hh * 16 + j]);
          }
          // diagonal m drained: the MMA warp may overwrite it for the next pass
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) ob_arrive(&acc_empty[m - 2]);
        }
        if (pass == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) re[j] = ldexp(v[j], er + __shfl_sync(0xffffffffu, ec_lane, j));
        } else {
          double2* orow = sp.out[g.cc] + (int64_t)row * sp.ld[g.cc];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = col0 + j;
            const int ecj = __shfl_sync(0xffffffffu, ec_lane, j);  // whole warp participates
            if (row < g.R && col < g.C) orow[col] = make_double2(re[j], ldexp(v[j], er + ecj));
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- launchers ----------------------------------------------------------------------------------
template <int S>
static cudaError_t stage_s(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1, cudaStream_t s) {
  const int ng = (int)p->oz_groups.size();
  int maxr = 0, maxc = 0;
  for (const auto& g : p->oz_groups) {
    maxr = std::max(maxr, g.nmt * OZ_BM);
    maxc = std::max(maxc, g.nnt * OZ_BN);
  }
  k3o_rows<S><<<dim3((maxr + 7) / 8, ng), 256, 0, s>>>(p->d_oz_groups, p->d_perm[0], p->d_perm[1], gk, p->chi[1], lk,
                                                       p->d_oa, p->d_oea);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k3o_cols<S><<<dim3((maxc + 255) / 256, ng), 256, 0, s>>>(p->d_oz_groups, p->d_perm[1], p->d_perm[2], gk1,
                                                            p->chi[2], p->d_ob, p->d_oeb);
  return cudaGetLastError();
}

cudaError_t launch_oz_stage(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1, cudaStream_t s) {
  if (p->oz_groups.empty()) return cudaSuccess;
  switch (p->oz_slices) {
    case 4: return stage_s<4>(p, gk, lk, gk1, s);
    case 5: return stage_s<5>(p, gk, lk, gk1, s);
    case 6: return stage_s<6>(p, gk, lk, gk1, s);
    case 7: return stage_s<7>(p, gk, lk, gk1, s);
    case 8: return stage_s<8>(p, gk, lk, gk1, s);
  }
  return cudaErrorInvalidValue;
}

template <int S, int STG>
static cudaError_t contract_st(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  const size_t smem = (size_t)STG * S * (OZ_A_TILE + OZ_B_TILE) + 8 * (2 * STG + 1 + S) + 16;
  cudaError_t e = cudaFuncSetAttribute(k4o_contract<S, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(p->oz_ntiles, p->sm_count);
  k4o_contract<S, STG><<<grid, OZ_THREADS, smem, s>>>(p->d_oz_groups, p->d_oz_tiles, (int)p->oz_ntiles, p->d_oa,
                                                      p->d_ob, p->d_oea, p->d_oeb, sp);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k4o_contract<S, STG>);
    fprintf(stderr, "k4o launch failed: %s regs=%d maxthreads=%d static_smem=%zu dyn_smem=%zu max_dyn=%d local=%zu\n",
            cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, smem,
            fa.maxDynamicSharedSizeBytes, fa.localSizeBytes);
  }
  return e;
}

// deepest TMA ring of half steps that fits in the 227 KB opt-in shared memory (S=6: 6, S=7: 5, S=8: 4)
template <int S>
static cudaError_t contract_s(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  constexpr int stage = S * (OZ_A_TILE + OZ_B_TILE);
  constexpr int limit = 227 * 1024 - 512;
  if constexpr (6 * stage <= limit) return contract_st<S, 6>(p, sp, s);
  else if constexpr (5 * stage <= limit) return contract_st<S, 5>(p, sp, s);
  else return contract_st<S, 4>(p, sp, s);
}

cudaError_t launch_oz_contract(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  if (p->oz_ntiles == 0) return cudaSuccess;
  switch (p->oz_slices) {
    case 4: return contract_s<4>(p, sp, s);
    case 5: return contract_s<5>(p, sp, s);
    case 6: return contract_s<6>(p, sp, s);
    case 7: return contract_s<7>(p, sp, s);
    case 8: return contract_s<8>(p, sp, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tn
