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
// [plane (Br, −Bi, Bi)][slice] for B, so one stage of K4O is ONE contiguous bulk copy per operand.
//
// Contraction (K4O). Persistent CTA per SM, 10 warps: warp 0 streams "half steps" (one A plane and one
// B plane of one K step, S slices each) with cp.async.bulk (TMA) into a 4–6 deep mbarrier ring; warp 1
// owns TMEM (512 columns = 8 slots of 64) and one thread issues tcgen05.mma.cta_group::1.kind::i8
// (M=128, N=64, K=32) into one int32 accumulator slot per diagonal m = p+q. A tile is two passes (Re, Im);
// pass P uses slots (S·P + i) mod 8, so it opens on slots freed long ago, and a diagonal whose slot is
// still being drained is deferred (its half steps stay in the ring and are replayed once the slot frees).
// The last half step commits each diagonal to its own slot_full barrier; warps 2–9 drain a slot with
// one tcgen05.ld.32x32b.x32, release it, and fold it into Σ_m D_m·2^{7(S+1−m)} (exact int64 for S ≤ 6,
// one rounding at the end; FP64 for S ≥ 7), scale by 2^{e_i+f_j} and store the Re / Im halves of P.
// Every int32 accumulator is exact: |D_m| ≤ 2·(m−1)·K·127² < 2^31 for K ≤ 2048 (OZ_KMAX, enforced).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tn_internal.cuh"

namespace tn {

// byte offset of element (r, k) (k < 32) inside one canonical rows×32 K-major tile
__host__ __device__ __forceinline__ int oz_canon(int r, int k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

// exact 2^e (bit-built when normal; ldexp covers the subnormal / overflow range)
__device__ __forceinline__ double oz_pow2(int e) {
  return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(e + 1023) << 52) : ldexp(1.0, e);
}

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

// ---- K3O: scales (one pass over the δ-allowed block) then slices (a second, L2-friendly pass) ------
// Row exponent of A (λk folded in): one warp per row, lanes across K.
__global__ void __launch_bounds__(256) k3o_row_exp(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_l,
                                                   const int32_t* __restrict__ perm_c, const double2* __restrict__ gk,
                                                   int64_t ld_gk, const double* __restrict__ lk, int32_t* __restrict__ oea) {
  const OzGroup g = groups[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= g.R) return;
  const double2* grow = gk + (int64_t)perm_l[g.row0 + r] * ld_gk;
  double mx = 0.0;
  for (int k = lane; k < g.K; k += 32) {
    const int32_t gc = perm_c[g.k0 + k];
    const double2 v = grow[gc];
    const double s = lk[gc];
    mx = fmax(mx, fmax(fabs(v.x * s), fabs(v.y * s)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) oea[g.ea_off + r] = mx > 0.0 ? ilogb(mx) + 1 : 0;
}

// Column exponent of B: 64 columns × 4 K quarters per CTA (coalesced rows), max-reduced in shared memory.
__global__ void __launch_bounds__(256) k3o_col_exp(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_c,
                                                   const int32_t* __restrict__ perm_r, const double2* __restrict__ gk1,
                                                   int64_t ld_gk1, int32_t* __restrict__ oeb) {
  __shared__ double red[4][64];
  const OzGroup g = groups[blockIdx.y];
  const int jj = threadIdx.x & 63, qk = threadIdx.x >> 6;
  const int j = blockIdx.x * 64 + jj;
  if (blockIdx.x * 64 >= g.C) return;  // CTA-uniform
  const bool valid = j < g.C;
  const int64_t pc = valid ? perm_r[g.col0 + j] : 0;
  double mx = 0.0;
  if (valid)
#pragma unroll 4
    for (int k = qk; k < g.K; k += 4) {
      const double2 v = gk1[(int64_t)perm_c[g.k0 + k] * ld_gk1 + pc];
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
  red[qk][jj] = mx;
  __syncthreads();
  if (qk == 0 && valid) {
    mx = fmax(fmax(red[0][jj], red[1][jj]), fmax(red[2][jj], red[3][jj]));
    oeb[g.eb_off + j] = mx > 0.0 ? ilogb(mx) + 1 : 0;
  }
}

// A slices of one (row tile, K step): thread = row of the 128-row tile, 32 K values, 2 planes × S slices.
// Stores: a warp's 32 rows form 4 complete 8-row core-matrix groups → contiguous 16-byte pieces.
template <int S>
__global__ void __launch_bounds__(128) k3o_rows(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_l,
                                                const int32_t* __restrict__ perm_c, const double2* __restrict__ gk,
                                                int64_t ld_gk, const double* __restrict__ lk,
                                                const int32_t* __restrict__ oea, int8_t* __restrict__ oa) {
  const OzGroup g = groups[blockIdx.y];
  const int mt = blockIdx.x / g.nkc, kc = blockIdx.x % g.nkc;
  if (mt >= g.nmt) return;
  const int rr = threadIdx.x, r = mt * OZ_BM + rr;
  const bool valid = r < g.R;
  const double2* grow = gk + (valid ? (int64_t)perm_l[g.row0 + r] * ld_gk : 0);
  const double scale = oz_pow2(-(valid ? oea[g.ea_off + r] : 0));  // exact: |x·2^−e| < 1
  int8_t* base = oa + g.a_off + (int64_t)(mt * g.nkc + kc) * (2 * S) * OZ_A_TILE;
#pragma unroll 1
  for (int hk = 0; hk < 2; ++hk) {
    double re[16], im[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = kc * OZ_BK + hk * 16 + i;
      re[i] = im[i] = 0.0;
      if (valid && k < g.K) {
        const int32_t gc = perm_c[g.k0 + k];
        const double2 v = grow[gc];
        const double sc = lk[gc] * scale;
        re[i] = v.x * sc;
        im[i] = v.y * sc;
      }
    }
    int8_t* b = base + oz_canon(rr, hk * 16);
    uint4 sl[S];
    slice16<S>(re, sl);
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(b + (int64_t)p * OZ_A_TILE) = sl[p];
    slice16<S>(im, sl);
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(b + (int64_t)(S + p) * OZ_A_TILE) = sl[p];
  }
}

// B slices of one (column tile, K step): thread = column of the 64-column tile; planes Br, −Bi, Bi.
template <int S>
__global__ void __launch_bounds__(256) k3o_cols(const OzGroup* __restrict__ groups, const int32_t* __restrict__ perm_c,
                                               const int32_t* __restrict__ perm_r, const double2* __restrict__ gk1,
                                               int64_t ld_gk1, const int32_t* __restrict__ oeb, int8_t* __restrict__ ob) {
  const OzGroup g = groups[blockIdx.y];
  const int nkq = (g.nkc + 3) >> 2;  // K steps in groups of 4 (one per 64-thread quarter)
  const int nt = blockIdx.x / nkq, kc = (blockIdx.x % nkq) * 4 + (threadIdx.x >> 6);
  if (nt >= g.nnt || kc >= g.nkc) return;
  const int jj = threadIdx.x & 63, j = nt * OZ_BN + jj;
  const bool valid = j < g.C;
  const int64_t pc = valid ? perm_r[g.col0 + j] : 0;
  const double scale = oz_pow2(-(valid ? oeb[g.eb_off + j] : 0));
  int8_t* base = ob + g.b_off + (int64_t)(nt * g.nkc + kc) * (3 * S) * OZ_B_TILE;
#pragma unroll 1
  for (int hk = 0; hk < 2; ++hk) {
    double re[16], im[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = kc * OZ_BK + hk * 16 + i;
      re[i] = im[i] = 0.0;
      if (valid && k < g.K) {
        const double2 v = gk1[(int64_t)perm_c[g.k0 + k] * ld_gk1 + pc];
        re[i] = v.x * scale;
        im[i] = v.y * scale;
      }
    }
    int8_t* b = base + oz_canon(jj, hk * 16);
    uint4 sl[S];
    slice16<S>(re, sl);  // plane 0: Br
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(b + (int64_t)p * OZ_B_TILE) = sl[p];
    slice16<S>(im, sl);  // plane 2: Bi
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(b + (int64_t)(2 * S + p) * OZ_B_TILE) = sl[p];
#pragma unroll
    for (int i = 0; i < 16; ++i) im[i] = -im[i];
    slice16<S>(im, sl);  // plane 1: −Bi
#pragma unroll
    for (int p = 0; p < S; ++p) *reinterpret_cast<uint4*>(b + (int64_t)(S + p) * OZ_B_TILE) = sl[p];
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
__device__ __forceinline__ bool ob_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
// suspending wait for the side warps (producer, epilogue): they share SM sub-partitions with the MMA
// issuer, so they must not burn issue slots polling (each try_wait may park the warp up to ~hint ns)
__device__ __forceinline__ void ob_sleep_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(s32(b)), "r"(parity), "r"(20000)
        : "memory");
  } while (!done);
}
// non-suspending poll (try_wait may park the thread for a system-dependent time before re-checking)
__device__ __forceinline__ void ob_spin(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
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
constexpr int OZ_SLOTS = 512 / OZ_BN;  // TMEM accumulator slots
// order in which a pass opens its diagonals m = 2..S+1: the two largest (most slice pairs) first, on the
// slots left free by the previous pass, then m = 2, 3, … in the order the epilogue frees them
__host__ __device__ constexpr int oz_diag(int S, int i) { return i == 0 ? S + 1 : i == 1 ? S : i; }

// One ring stage = one "half step": A plane h (S slices, 128×32 each) and B plane 2·pass + h (S slices,
// 64×32 each) of one K step of one tile; the Re pass pairs (Ar, Br), (Ai, −Bi), the Im pass (Ar, Bi),
// (Ai, Br). Small stages let the ring run 5–6 deep (the v1 ring of whole K steps was only 2 deep).
// D·2^E as int64 in one IMAD.WIDE (E ≤ 30) or one add into the high word (E ≥ 32; D·2^(E−32) fits int32
// because |D| ≤ 2(m−1)·Kp·127² < 2^26 for the m with E ≥ 32, i.e. m = 2 at S = 6).
// (E is a compile-time constant after unrolling; 7(S+1−m) ∈ {0, 7, …, 35} for S ≤ 6, never 31)
__device__ __forceinline__ int64_t oz_weighted(int32_t d, int E) {
  if (E <= 30) return (int64_t)d * (int64_t)(1 << E);
  return (int64_t)(d * (1 << (E - 32))) << 32;
}

template <int S>
__device__ __forceinline__ void oz_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile("{\n .reg .pred pp;\n setp.ne.b32 pp, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n" ::"r"(d),
               "l"(da), "l"(db), "r"(OZ_IDESC), "r"(acc));
}

template <int S, int OZ_STAGES>
__global__ void __launch_bounds__(OZ_THREADS, 1)  // 10 warps: ≤ 3 per SM sub-partition → ≤ 168 registers
    k4o_contract(const OzGroup* __restrict__ groups, const OzTile* __restrict__ tiles, int ntiles,
                 const int8_t* __restrict__ oa, const int8_t* __restrict__ ob, const int32_t* __restrict__ oea,
                 const int32_t* __restrict__ oeb, const SectorParams sp) {
  constexpr int A_HS = S * OZ_A_TILE, B_HS = S * OZ_B_TILE;   // one plane of one K step
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + OZ_STAGES * A_HS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + OZ_STAGES * B_HS);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* slot_full = empty + OZ_STAGES;       // per TMEM slot (64 columns): its diagonal is complete
  uint64_t* slot_empty = slot_full + OZ_SLOTS;   // per TMEM slot: the epilogue has drained it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(slot_empty + OZ_SLOTS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      ob_init(&full[s], 1);
      ob_init(&empty[s], 1);
    }
    for (int m = 0; m < OZ_SLOTS; ++m) {
      ob_init(&slot_full[m], 1);
      ob_init(&slot_empty[m], 8);  // the 8 epilogue warps
    }
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
        const int8_t* b_t = ob + g.b_off + (int64_t)td.nt * g.nkc * 3 * B_HS;
        for (int pass = 0; pass < 2; ++pass)
          for (int kc = 0; kc < g.nkc; ++kc)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              ob_sleep_wait(&empty[stage], phase ^ 1);
              ob_expect_tx(&full[stage], A_HS + B_HS);
              ob_bulk(sA + stage * A_HS, a_t + (int64_t)(kc * 2 + h) * A_HS, A_HS, &full[stage]);
              // B planes [Br, −Bi, Bi]: Re pass (Br, −Bi), Im pass (Bi, Br)
              const int bp = pass == 0 ? h : (h == 0 ? 2 : 0);
              ob_bulk(sB + stage * B_HS, b_t + (int64_t)(kc * 3 + bp) * B_HS, B_HS, &full[stage]);
              if (++stage == OZ_STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // TMEM = 8 slots of 64 columns; pass P keeps its S diagonal accumulators in slots (S·P + i) mod 8,
    // i = position of the diagonal in oz_diag (no accumulator double-buffer fits). A pass opens its
    // diagonals as their slots come free; a diagonal whose slot is still being drained is DEFERRED: its
    // half steps stay in the ring (not released) and are replayed for it once the slot frees, so the
    // MMA issue never stalls on the epilogue while operand stages remain.
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, slot_uses = 0;  // 2 bits per slot: parity of its use count
      int base = 0;
      constexpr uint32_t ALL = (1u << S) - 1;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int nhs = 2 * groups[tiles[t].g].nkc;
        for (int pass = 0; pass < 2; ++pass) {
          uint32_t col[S + 2];  // TMEM column of diagonal m (index m)
#pragma unroll
          for (int i = 0; i < S; ++i) col[oz_diag(S, i)] = (uint32_t)((base + i) & (OZ_SLOTS - 1)) * OZ_BN;
          // all slice pairs (p, m − p) of diagonal m against the half step in ring stage stg
          auto diag_on = [&](int m, int stg, bool fresh) {
            const uint64_t da = oz_desc(s32(sA + stg * A_HS)), db = oz_desc(s32(sB + stg * B_HS));
            const int pmin = m - S > 1 ? m - S : 1;
#pragma unroll
            for (int p = 1; p <= S; ++p) {
              const int q = m - p;
              if (q < 1 || q > S) continue;
              oz_mma<S>(tmem + col[m], da + (uint64_t)((p - 1) * OZ_A_TILE >> 4),
                        db + (uint64_t)((q - 1) * OZ_B_TILE >> 4), (fresh && p == pmin) ? 0u : 1u);
            }
          };
          auto commit = [&](uint64_t* bar) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
                         : "memory");
          };
          uint32_t acq = 0;           // bit i: diagonal oz_diag(S, i) owns its slot and has been started
          int held = 0;               // half steps of this pass kept in the ring (not yet released)
          const int st0 = stage;      // ring stage of the pass's first half step
          for (int hs = 0; hs < nhs; ++hs) {
            ob_wait(&full[stage], phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const bool last = hs == nhs - 1;
            if (acq != ALL) {
              // block for a slot only when deferring further would exhaust the ring, or at the last step
              const bool must = last || held + 2 > OZ_STAGES;
#pragma unroll
              for (int i = 0; i < S; ++i) {
                const int m = oz_diag(S, i);
                if (acq & (1u << i)) {
                  diag_on(m, stage, false);
                  continue;
                }
                const int sl = (base + i) & (OZ_SLOTS - 1);
                const uint32_t u = (slot_uses >> (2 * sl)) & 3u;
                bool ok = u == 0 || ob_test(&slot_empty[sl], (u - 1) & 1);
                if (!ok && must) {
                  ob_spin(&slot_empty[sl], (u - 1) & 1);
                  ok = true;
                }
                if (ok) {
                  slot_uses = (slot_uses & ~(3u << (2 * sl))) | ((u == 3 ? 2u : u + 1) << (2 * sl));
                  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                  int sx = st0;
                  for (int x = 0; x <= held; ++x) {  // replay the deferred half steps, then the current one
                    diag_on(m, sx, x == 0);
                    sx = sx + 1 == OZ_STAGES ? 0 : sx + 1;
                  }
                  acq |= 1u << i;
                }
              }
              if (acq == ALL) {
                int sx = st0;
                for (int x = 0; x <= held; ++x) {
                  commit(&empty[sx]);
                  sx = sx + 1 == OZ_STAGES ? 0 : sx + 1;
                }
                held = 0;
                if (last)
#pragma unroll
                  for (int i = 0; i < S; ++i) commit(&slot_full[(base + i) & (OZ_SLOTS - 1)]);
              } else {
                ++held;
              }
            } else if (last) {
              // last half step: diagonal by diagonal in slot order, each committed to its own slot_full
              // barrier so the epilogue drains slot i while the rest of the pass still runs
#pragma unroll
              for (int i = 0; i < S; ++i) {
                diag_on(oz_diag(S, i), stage, false);
                commit(&slot_full[(base + i) & (OZ_SLOTS - 1)]);
              }
              commit(&empty[stage]);
            } else {
              const uint64_t da = oz_desc(s32(sA + stage * A_HS)), db = oz_desc(s32(sB + stage * B_HS));
#pragma unroll
              for (int p = 1; p <= S; ++p)
#pragma unroll
                for (int q = 1; q <= S + 1 - p; ++q)
                  oz_mma<S>(tmem + col[p + q], da + (uint64_t)((p - 1) * OZ_A_TILE >> 4),
                            db + (uint64_t)((q - 1) * OZ_B_TILE >> 4), 1u);
              commit(&empty[stage]);
            }
            if (++stage == OZ_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          base = (base + S) & (OZ_SLOTS - 1);
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..9 ----------------
    const int quad = warp & 3;              // TMEM lanes 32·quad .. +31 (a warp's accessible quadrant)
    const int half = (warp - 2) >> 2;       // columns 32·half .. +31
    uint32_t slot_seen = 0;  // 2 bits per slot: parity of how many times it has been drained
    int ebase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const OzTile td = tiles[t];
      const OzGroup g = groups[td.g];
      const int row = td.mt * OZ_BM + quad * 32 + lane;
      const int col0 = td.nt * OZ_BN + half * 32;
      // exponents first (global loads off the accumulator critical path)
      const int er = row < g.R ? oea[g.ea_off + row] : 0;
      // lane j holds the exponent of column col0 + j (broadcast with shuffles below)
      const int ec_lane = (col0 + lane < g.C) ? oeb[g.eb_off + col0 + lane] : 0;
      for (int pass = 0; pass < 2; ++pass) {
        // S ≤ 6: exact int64 Horner Σ_m D_m·2^{7(S+1−m)} (< 2^59 for Kp ≤ 2048), one rounding at the end;
        // S ≥ 7 would overflow int64, so those accumulate Σ_m D_m·2^{−7m} in FP64.
        int64_t hacc[32];
        double v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          hacc[j] = 0;
          v[j] = 0.0;
        }
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const int m = oz_diag(S, i);
          const int sl = (ebase + i) & (OZ_SLOTS - 1);
          uint32_t r[32];
          const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)sl * OZ_BN + half * 32;
          {
            const uint32_t u = (slot_seen >> (2 * sl)) & 3u;
            ob_sleep_wait(&slot_full[sl], u & 1);
            slot_seen = (slot_seen & ~(3u << (2 * sl))) | ((u == 3 ? 2u : u + 1) << (2 * sl));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(ta));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // slot drained: the MMA warp may reuse it
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) ob_arrive(&slot_empty[sl]);
          if constexpr (S <= 6) {
#pragma unroll
            for (int j = 0; j < 32; ++j) hacc[j] += oz_weighted((int32_t)r[j], 7 * (S + 1 - m));
          } else {
            const double w = ldexp(1.0, -7 * m);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fma((double)(int32_t)r[j], w, v[j]);
          }
        }
        ebase = (ebase + S) & (OZ_SLOTS - 1);
        const double srow = oz_pow2(er - (S <= 6 ? 7 * (S + 1) : 0));
        // the Re pass stores the real halves, the Im pass the imaginary halves of the same 16-byte elements
        double* orow = reinterpret_cast<double*>(sp.sec[g.cc].out + (int64_t)row * sp.sec[g.cc].ld) + pass;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = col0 + j;
          const int ecj = __shfl_sync(0xffffffffu, ec_lane, j);  // whole warp participates
          double x;
          if constexpr (S <= 6) x = __ll2double_rn(hacc[j]) * srow * oz_pow2(ecj);
          else x = v[j] * srow * oz_pow2(ecj);
          if (row < g.R && col < g.C) orow[2 * col] = x;
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
static cudaError_t stage_s(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1, cudaStream_t s,
                           const int32_t* rowperm) {
  const int ng = (int)p->oz_groups.size();
  int maxr = 0, maxc = 0, maxa = 0, maxb = 0;
  for (const auto& g : p->oz_groups) {
    maxr = std::max(maxr, g.R);
    maxc = std::max(maxc, g.C);
    maxa = std::max(maxa, g.nmt * g.nkc);
    maxb = std::max(maxb, g.nnt * ((g.nkc + 3) / 4));
  }
  // the A chain (row exponents → A slices) and the B chain (column exponents → B slices) are independent:
  // the B chain runs on an auxiliary stream beside the A chain
  AuxStreams* aux = nullptr;
  cudaError_t e = aux_streams(s, &aux);
  if (e == cudaSuccess) e = cudaEventRecord(aux->fork, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(aux->st[0], aux->fork, 0);
  if (e != cudaSuccess) return e;
  cudaStream_t sb = aux->st[0];
  if (maxc > 0) k3o_col_exp<<<dim3((maxc + 63) / 64, ng), 256, 0, sb>>>(p->d_oz_groups, p->d_perm[1], p->d_colperm,
                                                                          gk1, p->chi[2], p->d_oeb);
  k3o_cols<S><<<dim3(maxb, ng), 4 * OZ_BN, 0, sb>>>(p->d_oz_groups, p->d_perm[1], p->d_colperm, gk1, p->chi[2], p->d_oeb,
                                                p->d_ob);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(aux->join[0], sb)) != cudaSuccess) return e;
  if (maxr > 0) k3o_row_exp<<<dim3((maxr + 7) / 8, ng), 256, 0, s>>>(p->d_oz_groups, rowperm, p->d_perm[1], gk,
                                                                     p->chi[1], lk, p->d_oea);
  k3o_rows<S><<<dim3(maxa, ng), OZ_BM, 0, s>>>(p->d_oz_groups, rowperm, p->d_perm[1], gk, p->chi[1], lk, p->d_oea,
                                               p->d_oa);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaStreamWaitEvent(s, aux->join[0], 0);
}

cudaError_t launch_oz_stage(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1, cudaStream_t s,
                            const int32_t* rowperm) {
  if (p->oz_groups.empty()) return cudaSuccess;
  switch (p->oz_slices) {
    case 4: return stage_s<4>(p, gk, lk, gk1, s, rowperm);
    case 5: return stage_s<5>(p, gk, lk, gk1, s, rowperm);
    case 6: return stage_s<6>(p, gk, lk, gk1, s, rowperm);
    case 7: return stage_s<7>(p, gk, lk, gk1, s, rowperm);
    case 8: return stage_s<8>(p, gk, lk, gk1, s, rowperm);
  }
  return cudaErrorInvalidValue;
}

template <int S, int STG>
static cudaError_t contract_st(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  const size_t smem = (size_t)STG * S * (OZ_A_TILE + OZ_B_TILE) + 8 * (2 * STG + 2 * OZ_SLOTS) + 16;
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
