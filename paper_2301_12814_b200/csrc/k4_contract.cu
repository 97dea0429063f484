// K4 — grouped block-sparse complex contraction on the FP64 tensor pipe (DMMA.8x8x4).
//
// For every center charge c_c with a non-empty segment ("without the U and λ value
// lookup, this is exactly the same as matrix multiplication"):
//   P_{c_c} = A_{c_c} · B_{c_c}       (R_{c_c} × K_{c_c}) · (K_{c_c} × C_{c_c}), complex128
// P_{c_c} has exactly the shape and index set of Θ(c_c), so it is written straight
// into the caller's Θ(c_c) buffer; K5 then applies U along the charge axis in place.
//
// B200 design (DESIGN.md §4 "K4"): sm_100a has no tcgen05 FP64 MMA (`kind::f64` does not exist),
// so the FP64 tensor path is the warp-level DMMA.8x8x4 (mma.sync.m8n8k4.f64), measured at 37.2
// TFLOP/s. A persistent grid (one CTA per SM) walks a heavy-first tile list; one producer warp
// streams each 64×32 operand stage (two 64×16 chunks) with a single cp.async.bulk (TMA 1-D) copy per
// operand into a 3-deep mbarrier ring; eight consumer warps (2×4, 32×16 complex outputs each) read fragments with
// conflict-free 128-bit LDS (K3 wrote the panels in fragment order). The complex product uses the
// 3-multiplication (Gauss) form, 3 real DMMAs per complex 8×8×4 step instead of 4:
//   T1 = Ar·Br, T2 = Ai·Bi, T3 = (Ar+Ai)·(Br+Bi);  Re = T1 − T2,  Im = T3 − T1 − T2
// (error bound ~ eps·|Ar+Ai||Br+Bi| per term, same order as the 4-product form).
#include <cstdlib>

#include "k4_device.cuh"

namespace tn {

// One ring stage of a warp's 32×16 outputs: MV of its four 8-row m-subtiles and NV of its two 8-column
// n-subtiles hold valid rows / columns (the rest is tile padding: its DMMAs are skipped — at a shard's or a
// group's ragged edge up to 56 of 64 rows are padding, and the DMMA pipe is what bounds K4).
// One 8×8×4 complex step: the Gauss sums first, then all T1/T2 products (which do not need them), then the T3
// products — every DMMA is issued well after the DADD that feeds it.
template <int MV, int NV, int KSTEPS>
__device__ __forceinline__ void k4_stage(double (&acc)[4][2][6], const double2* __restrict__ As,
                                         const double2* __restrict__ Bs, int nks) {
  auto kstep = [&](int ks) {
    double2 a[MV], b[NV];
#pragma unroll
    for (int mi = 0; mi < MV; ++mi) a[mi] = As[ks * 256 + mi * 32];
#pragma unroll
    for (int ni = 0; ni < NV; ++ni) b[ni] = Bs[ks * 256 + ni * 32];
    double asum[MV], bsum[NV];
#pragma unroll
    for (int ni = 0; ni < NV; ++ni) bsum[ni] = b[ni].x + b[ni].y;
#pragma unroll
    for (int mi = 0; mi < MV; ++mi) asum[mi] = a[mi].x + a[mi].y;
#pragma unroll
    for (int mi = 0; mi < MV; ++mi)
#pragma unroll
      for (int ni = 0; ni < NV; ++ni) {
        double* c = acc[mi][ni];
        dmma(c[0], c[1], a[mi].x, b[ni].x);  // T1 += Ar·Br
        dmma(c[2], c[3], a[mi].y, b[ni].y);  // T2 += Ai·Bi
      }
#pragma unroll
    for (int mi = 0; mi < MV; ++mi)
#pragma unroll
      for (int ni = 0; ni < NV; ++ni) dmma(acc[mi][ni][4], acc[mi][ni][5], asum[mi], bsum[ni]);  // T3
  };
  if (nks == KSTEPS) {  // full stage: no guards, so the fragment loads of step ks+1 can overlap step ks
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) kstep(ks);
  } else {
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks)
      if (ks < nks) kstep(ks);
  }
}

template <int STAGES, int CPS>  // CPS: BK-chunks per ring stage (one bulk copy per operand per stage)
__global__ void __launch_bounds__(K4_THREADS, 1)
    k4_contract(const GroupDesc* __restrict__ groups, const TileDesc* __restrict__ tiles, int ntiles,
                const double2* __restrict__ ap, const double2* __restrict__ bp, const SectorParams sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  double2* sA = reinterpret_cast<double2*>(smem);
  constexpr int SCH = CPS * CHUNK, SBK = CPS * BK;  // elements / K per stage
  double2* sB = sA + STAGES * SCH;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * SCH);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], K4_CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == K4_CONSUMER_WARPS) {
    // ---------------- producer: one elected lane streams A/B chunks ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      TileDesc pd_next = tiles[blockIdx.x];
      GroupDesc pg_next = groups[pd_next.g];
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileDesc td = pd_next;
        const GroupDesc g = pg_next;
        if (t + (int)gridDim.x < ntiles) {
          pd_next = tiles[t + gridDim.x];
          pg_next = groups[pd_next.g];
        }
        const double2* a = ap + g.a_off + (int64_t)td.mt * BM * g.K4;
        const double2* b = bp + g.b_off + (int64_t)td.nt * BN * g.K4;
        for (int kc = 0; kc * SBK < g.K4; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t kcnt = (uint32_t)min(SBK, g.K4 - kc * SBK);
          const uint32_t bytes = kcnt * BM * (uint32_t)sizeof(double2);
          mbar_expect_tx(&full[stage], 2 * bytes);
          bulk_g2s(sA + stage * SCH, a + (int64_t)kc * SCH, bytes, &full[stage]);
          bulk_g2s(sB + stage * SCH, b + (int64_t)kc * SCH, bytes, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: 2×4 warps, 32×16 complex outputs each ----------------
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  // tile / group descriptors of the NEXT tile are loaded during the current one (their global-load
  // latency would otherwise stall all consumer warps at every tile start)
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
    double acc[4][2][6];  // [mi][ni][T1 0,1 | T2 0,1 | T3 0,1]
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[mi][ni][q] = 0.0;

    // valid 8-row / 8-column subtiles of this warp's 32×16 outputs (full tiles: 4 and 2)
    const int rows_w = g.R - (td.mt * BM + wm * 32), cols_w = g.C - (td.nt * BN + wn * 16);
    const int mv = rows_w <= 0 ? 0 : min(4, (rows_w + 7) >> 3);
    const int nv = cols_w <= 0 ? 0 : min(2, (cols_w + 7) >> 3);
    const int shape = (mv == 0 || nv == 0) ? 0 : mv * 2 + nv - 2;   // 1..8; 8 = full
    for (int kc = 0; kc * SBK < g.K4; ++kc) {
      mbar_wait(&full[stage], phase);
      const int nks = min(SBK, g.K4 - kc * SBK) >> 2;
      const double2* As = sA + stage * SCH + wm * 128 + lane;
      const double2* Bs = sB + stage * SCH + wn * 64 + lane;
      constexpr int KS = 4 * CPS;
      switch (shape) {
        case 8: k4_stage<4, 2, KS>(acc, As, Bs, nks); break;
        case 7: k4_stage<4, 1, KS>(acc, As, Bs, nks); break;
        case 6: k4_stage<3, 2, KS>(acc, As, Bs, nks); break;
        case 5: k4_stage<3, 1, KS>(acc, As, Bs, nks); break;
        case 4: k4_stage<2, 2, KS>(acc, As, Bs, nks); break;
        case 3: k4_stage<2, 1, KS>(acc, As, Bs, nks); break;
        case 2: k4_stage<1, 2, KS>(acc, As, Bs, nks); break;
        case 1: k4_stage<1, 1, KS>(acc, As, Bs, nks); break;
        default: break;  // no valid output in this warp's quarter of the tile
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // epilogue: P tile → Θ(c_c) slab (row-major, ld = C_{c_c}); lane owns rows gq, cols 2tq, 2tq+1
    double2* out = sp.sec[g.cc].out;
    const int ld = sp.sec[g.cc].ld;
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
  }
}

template <int STAGES, int CPS>
static cudaError_t contract_cfg(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  const size_t smem = (size_t)STAGES * CPS * CHUNK * sizeof(double2) * 2 + 2 * STAGES * sizeof(uint64_t);
  // set on every launch (microseconds): the attribute is per device, and a process may drive several
  cudaError_t e =
      cudaFuncSetAttribute(k4_contract<STAGES, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(p->ntiles, (int64_t)p->sm_count);
  k4_contract<STAGES, CPS><<<(unsigned)grid, K4_THREADS, smem, s>>>(p->d_groups, p->d_tiles, (int)p->ntiles,
                                                                     p->d_apanel, p->d_bpanel, sp);
  return cudaGetLastError();
}

cudaError_t launch_contract(const tn_plan* p, const SectorParams& sp, cudaStream_t s) {
  if (p->ntiles == 0) return cudaSuccess;
  // 3 stages of 2 chunks (32-deep K per barrier round trip) by default: 2.533 vs 2.558 ms for 6 stages of
  // one chunk at config 3, 18.88 vs 19.03 ms at config 4 (TN_K4_CPS=1 selects the latter)
  static const int cps = getenv("TN_K4_CPS") ? atoi(getenv("TN_K4_CPS")) : 2;
  if (cps == 1) return contract_cfg<K4_STAGES, 1>(p, sp, s);
  return contract_cfg<3, 2>(p, sp, s);
}

}  // namespace tn
