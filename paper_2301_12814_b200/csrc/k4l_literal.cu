// K3L + K4L — the paper's own Θ(c) kernel shape, kept as an ABLATION:
// "one GEMM per Θ(c) with U lookup" ("We adopt all aforementioned techniques in
// our GPU kernel for obtaining Θ(c^k), with the added complexity of complex number support and U matrix
// value look-up based on charges"). Selected with tn_plan_set_contraction(plan, TN_CONTRACT_PAPER_LITERAL).
//
// For every sector c, Θ(c) is ONE GEMM over the concatenated centre segments c_c ∈ [c−d+1, c+d−1]:
//   Θ(c)[α,β] = λl λr Σ_{c_c} U_{c_l−c_r}[c_l−c][c_l−c_c] Σ_{α_k ∈ seg(c_c)} Γk[α,α_k] λk Γk1[α_k,β]
// The U weight depends on the row charge, the column charge and c_c, so it is applied per element at
// every c_c segment boundary of the K loop (segments zero-padded to the 16-wide K chunk; δ-forbidden
// operand entries staged as zeros — they are never read from Γ). Same DMMA.8x8x4 3M mainloop, TMA-bulk
// ring and fragment-ordered panels as K4; no K5. The work is Σ_c R_c·C_c·K_c instead of the product-once
// Σ_{c_c} R·C·K + mix (12× more at config 3, SURVEY.md §8(d) F_paperA): the ablation measures what the
// reformulation buys on the same hardware path.
#include "k4_device.cuh"

namespace tn {

struct LitSeg {             // one centre segment inside sector s's K range
  int32_t cc, kdst, ksrc, len;   // centre charge, first padded K index, first sorted centre position, bonds
};

// A_s[r][k] / B_s[k][n] in K3's fragment order (see k3_stage.cu), K4 = padded K of the sector
__global__ void __launch_bounds__(256) k3l_stage_a(const LitSector* __restrict__ secs, const LitSeg* __restrict__ segs,
                                                   const int32_t* __restrict__ perm_l, const int32_t* __restrict__ qs_l,
                                                   const int32_t* __restrict__ perm_c, const double2* __restrict__ gk,
                                                   int64_t ld_gk, const double* __restrict__ lk, int d,
                                                   double2* __restrict__ ap) {
  const LitSector S = secs[blockIdx.y];
  const int64_t tile_elems = (int64_t)BM * S.K4;
  const int64_t total = tile_elems * S.nmt;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t mt = e / tile_elems;
    const int64_t rem = e - mt * tile_elems;
    const int kc = (int)(rem >> 10), w = (int)(rem & 1023);
    const int ks = w >> 8, wm = (w >> 7) & 1, mi = (w >> 5) & 3, lane = w & 31;
    const int64_t row = mt * BM + wm * 32 + mi * 8 + (lane >> 2);
    const int k = kc * BK + ks * 4 + (lane & 3);
    double2 v = make_double2(0.0, 0.0);
    if (row < S.R) {
      int sg = 0;
      while (sg + 1 < S.nseg && segs[S.seg0 + sg + 1].kdst <= k) ++sg;
      const LitSeg g = segs[S.seg0 + sg];
      const int kk = k - g.kdst;
      const int dq = qs_l[S.row0 + row] - g.cc;  // j_k = c_l − c_c must lie in [0, d−1]
      if (kk < g.len && dq >= 0 && dq <= d - 1) {
        const int32_t gc = perm_c[g.ksrc + kk];
        const double2 x = gk[(int64_t)perm_l[S.row0 + row] * ld_gk + gc];
        const double s = lk[gc];
        v = make_double2(x.x * s, x.y * s);
      }
    }
    ap[S.a_off + e] = v;
  }
}

__global__ void __launch_bounds__(256) k3l_stage_b(const LitSector* __restrict__ secs, const LitSeg* __restrict__ segs,
                                                   const int32_t* __restrict__ perm_c, const int32_t* __restrict__ perm_r,
                                                   const int32_t* __restrict__ qs_r, const double2* __restrict__ gk1,
                                                   int64_t ld_gk1, int d, double2* __restrict__ bp) {
  const LitSector S = secs[blockIdx.y];
  const int64_t tile_elems = (int64_t)BN * S.K4;
  const int64_t total = tile_elems * S.nnt;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nt = e / tile_elems;
    const int64_t rem = e - nt * tile_elems;
    const int kc = (int)(rem >> 10), w = (int)(rem & 1023);
    const int ks = w >> 8, wn = (w >> 7) & 1, ni = (w >> 5) & 3, lane = w & 31;
    const int64_t col = nt * BN + wn * 32 + ni * 8 + (lane >> 2);
    const int k = kc * BK + ks * 4 + (lane & 3);
    double2 v = make_double2(0.0, 0.0);
    if (col < S.C) {
      int sg = 0;
      while (sg + 1 < S.nseg && segs[S.seg0 + sg + 1].kdst <= k) ++sg;
      const LitSeg g = segs[S.seg0 + sg];
      const int kk = k - g.kdst;
      const int dq = g.cc - qs_r[S.col0 + col];  // j_{k+1} = c_c − c_r must lie in [0, d−1]
      if (kk < g.len && dq >= 0 && dq <= d - 1)
        v = gk1[(int64_t)perm_c[g.ksrc + kk] * ld_gk1 + perm_r[S.col0 + col]];
    }
    bp[S.b_off + e] = v;
  }
}

template <int STAGES>
__global__ void __launch_bounds__(K4_THREADS, 1)
    k4l_contract(const LitSector* __restrict__ secs, const LitSeg* __restrict__ segs, const TileDesc* __restrict__ tiles,
                 int ntiles, const double2* __restrict__ ap, const double2* __restrict__ bp,
                 const int32_t* __restrict__ qs_l, const int32_t* __restrict__ qs_r, const int32_t* __restrict__ perm_l,
                 const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
                 const double2* __restrict__ U, const SectorParams sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  double2* sA = reinterpret_cast<double2*>(smem);
  double2* sB = sA + STAGES * CHUNK;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * CHUNK);
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
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileDesc td = tiles[t];
        const LitSector S = secs[td.g];
        const double2* a = ap + S.a_off + (int64_t)td.mt * BM * S.K4;
        const double2* b = bp + S.b_off + (int64_t)td.nt * BN * S.K4;
        for (int kc = 0; kc * BK < S.K4; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t bytes = (uint32_t)(BK * BM * sizeof(double2));
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
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, tq = lane & 3;
  const int d = sp.d;
  int stage = 0;
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const TileDesc td = tiles[t];
    const LitSector S = secs[td.g];
    const int c = S.c;
    int cl[4], cr[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int row = td.mt * BM + wm * 32 + mi * 8 + gq;
      cl[mi] = row < S.R ? qs_l[S.row0 + row] : -1;
    }
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = td.nt * BN + wn * 16 + ni * 8 + 2 * tq + h;
        cr[ni * 2 + h] = col < S.C ? qs_r[S.col0 + col] : -1;
      }
    double th[4][2][4];   // Θ accumulators: [mi][ni][re0, im0, re1, im1]
    double acc[4][2][6];  // one segment's P: Gauss T1, T2, T3 per element pair
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
#pragma unroll
        for (int q = 0; q < 4; ++q) th[mi][ni][q] = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[mi][ni][q] = 0.0;
      }
    int sg = 0;
    for (int kc = 0; kc * BK < S.K4; ++kc) {
      mbar_wait(&full[stage], phase);
      const double2* As = sA + stage * CHUNK + wm * 128 + lane;
      const double2* Bs = sB + stage * CHUNK + wn * 64 + lane;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
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
            double* cc = acc[mi][ni];
            dmma(cc[0], cc[1], a[mi].x, b[ni].x);
            dmma(cc[2], cc[3], a[mi].y, b[ni].y);
            dmma(cc[4], cc[5], asum, bsum[ni]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      // end of a centre segment: Θ += U_{c_l−c_r}[c_l−c][c_l−c_c] · P, element by element (the paper's lookup)
      const bool seg_end = (kc + 1) * BK >= S.K4 || (sg + 1 < S.nseg && segs[S.seg0 + sg + 1].kdst <= (kc + 1) * BK);
      if (seg_end) {
        const int cc = segs[S.seg0 + sg].cc;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double* q = acc[mi][ni];
              const double pr = q[h] - q[2 + h], pi = q[4 + h] - q[h] - q[2 + h];
              const int l = cl[mi], r = cr[ni * 2 + h];
              double2 w = make_double2(0.0, 0.0);
              if (l >= 0 && r >= 0 && l - cc >= 0 && l - cc <= d - 1 && cc - r >= 0 && cc - r <= d - 1 &&
                  l - c >= 0 && l - c <= d - 1 && c - r >= 0 && c - r <= d - 1) {
                const int n = l - r, nlo = max(0, n - d + 1), sn = min(n, d - 1) - nlo + 1;
                w = __ldg(U + sp.ustart[n] + (l - c - nlo) * sn + (l - cc - nlo));
              }
              th[mi][ni][2 * h] += w.x * pr - w.y * pi;
              th[mi][ni][2 * h + 1] += w.x * pi + w.y * pr;
            }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[mi][ni][q] = 0.0;
        ++sg;
      }
    }
    double2* out = sp.sec[c].out;
    const int ld = sp.sec[c].ld;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int row = td.mt * BM + wm * 32 + mi * 8 + gq;
      if (row >= S.R) continue;
      const double sl = ll[perm_l[S.row0 + row]];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = td.nt * BN + wn * 16 + ni * 8 + 2 * tq + h;
          if (col >= S.C) continue;
          const double s = sl * lr[perm_r[S.col0 + col]];
          out[(int64_t)row * ld + col] = make_double2(th[mi][ni][2 * h] * s, th[mi][ni][2 * h + 1] * s);
        }
    }
  }
}

// ---- plan side ----
tn_status build_literal(tn_plan* p) {
  const int N = p->N, d = p->d;
  const auto& oc = p->off[1];
  std::vector<LitSector>& secs = p->lit_secs;
  std::vector<LitSeg> segs;
  std::vector<TileDesc>& tiles = p->h_lit_tiles;
  secs.clear();
  tiles.clear();
  int64_t a_off = 0, b_off = 0;
  p->lit_flops = 0;
  for (int c = 0; c <= N; ++c) {
    if (p->lR[c] == 0 || p->C[c] == 0) continue;
    LitSector S{};
    S.c = c;
    S.row0 = p->lrow0[c];
    S.col0 = p->col0[c];
    S.R = (int32_t)p->lR[c];
    S.C = (int32_t)p->C[c];
    S.seg0 = (int32_t)segs.size();
    int32_t k = 0;
    for (int cc = std::max(0, c - d + 1); cc <= std::min(N, c + d - 1); ++cc) {
      const int32_t len = oc[cc + 1] - oc[cc];
      if (len == 0) continue;
      segs.push_back(LitSeg{cc, k, oc[cc], len});
      k += (len + BK - 1) / BK * BK;
    }
    S.nseg = (int32_t)segs.size() - S.seg0;
    if (S.nseg == 0) continue;
    S.K4 = k;
    S.nmt = (S.R + BM - 1) / BM;
    S.nnt = (S.C + BN - 1) / BN;
    S.a_off = a_off;
    S.b_off = b_off;
    a_off += (int64_t)S.nmt * BM * S.K4;
    b_off += (int64_t)S.nnt * BN * S.K4;
    p->lit_flops += 8 * (int64_t)S.nmt * BM * (int64_t)S.nnt * BN * S.K4;
    secs.push_back(S);
  }
  for (size_t i = 0; i < secs.size(); ++i)
    for (int mt = 0; mt < secs[i].nmt; ++mt)
      for (int nt = 0; nt < secs[i].nnt; ++nt) tiles.push_back(TileDesc{(int32_t)i, mt, nt, 0});
  std::stable_sort(tiles.begin(), tiles.end(), [&](const TileDesc& x, const TileDesc& y) { return secs[x.g].K4 > secs[y.g].K4; });
  if (p->blk_lit) {
    if (cudaEventSynchronize(p->ev_fence) != cudaSuccess) cudaGetLastError();   // last use (any stream)
    pool_release(p->blk_lit, nullptr, false);
    p->blk_lit = nullptr;
  }
  struct Cw {
    size_t off = 0;
    size_t take(size_t b) {
      const size_t o = off;
      off += (b + 255) & ~(size_t)255;
      return o;
    }
  } cw;
  const size_t o_s = cw.take(secs.size() * sizeof(LitSector)), o_g = cw.take(segs.size() * sizeof(LitSeg));
  const size_t o_t = cw.take(tiles.size() * sizeof(TileDesc));
  const size_t o_a = cw.take((size_t)a_off * 16), o_b = cw.take((size_t)b_off * 16);
  cudaError_t aerr = cudaSuccess;
  p->blk_lit = pool_alloc(std::max<size_t>(cw.off, 256), &aerr);
  if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (literal workspace)");
  char* base = static_cast<char*>(p->blk_lit);
  p->d_lit_secs = reinterpret_cast<LitSector*>(base + o_s);
  p->d_lit_segs = base + o_g;
  p->d_lit_tiles = reinterpret_cast<TileDesc*>(base + o_t);
  p->d_lit_a = reinterpret_cast<double2*>(base + o_a);
  p->d_lit_b = reinterpret_cast<double2*>(base + o_b);
  p->lit_ntiles = (int64_t)tiles.size();
  p->h_lit_segs.assign(reinterpret_cast<const char*>(segs.data()),
                       reinterpret_cast<const char*>(segs.data()) + segs.size() * sizeof(LitSeg));
  auto up = [&](void* dst, const void* src, size_t n) {
    return n ? cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, p->plan_stream) : cudaSuccess;
  };
  cudaError_t e = up(p->d_lit_secs, secs.data(), secs.size() * sizeof(LitSector));
  if (e == cudaSuccess) e = up(p->d_lit_segs, p->h_lit_segs.data(), p->h_lit_segs.size());
  if (e == cudaSuccess) e = up(p->d_lit_tiles, tiles.data(), tiles.size() * sizeof(TileDesc));
  if (e == cudaSuccess) e = cudaEventRecord(p->ev_ready, p->plan_stream);
  return cuda_check(e, "literal tables upload");
}

cudaError_t launch_literal(const tn_plan* p, const SectorParams& sp, const double2* gk, const double* lk,
                           const double2* gk1, const double* ll, const double* lr, const double2* U, cudaStream_t s,
                           cudaEvent_t mid) {
  const int ns = (int)p->lit_secs.size();
  if (ns == 0) return cudaEventRecord(mid, s);
  int64_t amax = 0, bmax = 0;
  for (const auto& S : p->lit_secs) {
    amax = std::max<int64_t>(amax, (int64_t)BM * S.K4 * S.nmt);
    bmax = std::max<int64_t>(bmax, (int64_t)BN * S.K4 * S.nnt);
  }
  auto blocks = [&](int64_t total) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4096)); };
  const LitSeg* segs = reinterpret_cast<const LitSeg*>(p->d_lit_segs);
  k3l_stage_a<<<dim3(blocks(amax), ns), 256, 0, s>>>(p->d_lit_secs, segs, p->d_perm[0], p->d_qs[0], p->d_perm[1], gk,
                                                     p->chi[1], lk, p->d, p->d_lit_a);
  k3l_stage_b<<<dim3(blocks(bmax), ns), 256, 0, s>>>(p->d_lit_secs, segs, p->d_perm[1], p->d_perm[2], p->d_qs[2], gk1,
                                                     p->chi[2], p->d, p->d_lit_b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if ((e = cudaEventRecord(mid, s)) != cudaSuccess) return e;
  constexpr int STAGES = K4_STAGES;
  const size_t smem = (size_t)STAGES * CHUNK * sizeof(double2) * 2 + 2 * STAGES * sizeof(uint64_t);
  e = cudaFuncSetAttribute(k4l_contract<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(p->lit_ntiles, (int64_t)p->sm_count);
  k4l_contract<STAGES><<<(unsigned)grid, K4_THREADS, smem, s>>>(p->d_lit_secs, segs, p->d_lit_tiles, (int)p->lit_ntiles,
                                                                 p->d_lit_a, p->d_lit_b, p->d_qs[0], p->d_qs[2],
                                                                 p->d_perm[0], p->d_perm[2], ll, lr, U, sp);
  return cudaGetLastError();
}

}  // namespace tn
