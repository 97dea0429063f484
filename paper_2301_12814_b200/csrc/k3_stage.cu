// K3 — operand staging for the grouped contraction (sorted, padded bonds;
// BASELINE.json north_star item (3): "λ^{[k]} scaling fused into the operand load").
//
// For each center charge c_c (one "group"):
//   A_{c_c}[r][k] = Γk[perm_l[row0+r]][perm_c[k0+k]] · λk[perm_c[k0+k]]   (rows: Θ(c_c)'s rows)
//   B_{c_c}[k][n] = Γk1[perm_c[k0+k]][perm_r[col0+n]]                       (cols: Θ(c_c)'s cols)
// (pair plans pass per-group gathered row / column lists in place of perm_l / perm_r, tn_pair.cu)
// for k in seg_c(c_c). Only δ-allowed blocks of Γ are read. Panels are written in the
// exact DMMA fragment order the K4 consumer warps read, zero-padded to 64-row/col tiles and to a
// multiple of 4 in K (the "empty bonds" of PAPER.md:92), so one K4 chunk is a single contiguous
// cp.async.bulk copy. Chunk layout (complex elements, kc = 16-wide K chunk):
//   A: [mt][kc][ks(4)][wm(2)][mi(4)][lane(32)]  row = 32wm + 8mi + lane/4, k = 16kc + 4ks + lane%4
//   B: [nt][kc][ks(4)][wn(2)][ni(4)][lane(32)]  col = 32wn + 8ni + lane/4, k = 16kc + 4ks + lane%4
// A partial last chunk (K4 − 16kc < 16) is a prefix of the full layout (ks outermost).
#include "tn_internal.cuh"

namespace tn {

__global__ void __launch_bounds__(256) k3_stage_a(const GroupDesc* __restrict__ groups,
                                                  const int32_t* __restrict__ perm_l,
                                                  const int32_t* __restrict__ perm_c,
                                                  const double2* __restrict__ gk, int64_t ld_gk,
                                                  const double* __restrict__ lk, double2* __restrict__ ap) {
  const GroupDesc g = groups[blockIdx.y];
  const int64_t tile_elems = (int64_t)BM * g.K4;
  const int64_t total = tile_elems * g.nmt;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t mt = e / tile_elems;
    const int64_t rem = e - mt * tile_elems;
    const int kc = (int)(rem >> 10), w = (int)(rem & 1023);
    const int ks = w >> 8, wm = (w >> 7) & 1, mi = (w >> 5) & 3, lane = w & 31;
    const int64_t row = mt * BM + wm * 32 + mi * 8 + (lane >> 2);
    const int k = kc * BK + ks * 4 + (lane & 3);
    double2 v = make_double2(0.0, 0.0);
    if (row < g.R && k < g.K) {
      const int64_t a = perm_l[g.row0 + row];
      const int32_t gc = perm_c[g.k0 + k];
      const double2 x = gk[a * ld_gk + gc];
      const double s = lk[gc];
      v = make_double2(x.x * s, x.y * s);
    }
    ap[g.a_off + e] = v;
  }
}

__global__ void __launch_bounds__(256) k3_stage_b(const GroupDesc* __restrict__ groups,
                                                  const int32_t* __restrict__ perm_c,
                                                  const int32_t* __restrict__ perm_r,
                                                  const double2* __restrict__ gk1, int64_t ld_gk1,
                                                  double2* __restrict__ bp) {
  const GroupDesc g = groups[blockIdx.y];
  const int64_t tile_elems = (int64_t)BN * g.K4;
  const int64_t total = tile_elems * g.nnt;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nt = e / tile_elems;
    const int64_t rem = e - nt * tile_elems;
    const int kc = (int)(rem >> 10), w = (int)(rem & 1023);
    const int ks = w >> 8, wn = (w >> 7) & 1, ni = (w >> 5) & 3, lane = w & 31;
    const int64_t col = nt * BN + wn * 32 + ni * 8 + (lane >> 2);
    const int k = kc * BK + ks * 4 + (lane & 3);
    double2 v = make_double2(0.0, 0.0);
    if (col < g.C && k < g.K) {
      const int64_t r = perm_c[g.k0 + k];
      v = gk1[r * ld_gk1 + perm_r[g.col0 + col]];
    }
    bp[g.b_off + e] = v;
  }
}

cudaError_t launch_stage(const tn_plan* p, const double2* gk, const double* lk, const double2* gk1,
                         cudaStream_t s, const int32_t* rowperm) {
  const int ng = (int)p->groups.size();
  if (ng == 0) return cudaSuccess;
  int64_t amax = 0, bmax = 0;
  for (const auto& g : p->groups) {
    amax = std::max<int64_t>(amax, (int64_t)BM * g.K4 * g.nmt);
    bmax = std::max<int64_t>(bmax, (int64_t)BN * g.K4 * g.nnt);
  }
  const int64_t target = (int64_t)p->sm_count * 8;  // blocks in flight across all groups
  auto blocks = [&](int64_t total) {
    int64_t b = (total + 255) / 256;
    int64_t cap = std::max<int64_t>(1, target * 4 / ng);
    return (unsigned)std::max<int64_t>(1, std::min(b, cap));
  };
  // the A and B panels are disjoint: stage B on an auxiliary stream beside A (both HBM-bound, they share the
  // bandwidth but overlap each other's launch tails)
  AuxStreams* aux = nullptr;
  cudaError_t e = aux_streams(s, &aux);
  if (e == cudaSuccess) e = cudaEventRecord(aux->fork, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(aux->st[0], aux->fork, 0);
  if (e != cudaSuccess) return e;
  k3_stage_b<<<dim3(blocks(bmax), ng), 256, 0, aux->st[0]>>>(p->d_groups, p->d_perm[1], p->d_colperm, gk1,
                                                              p->chi[2], p->d_bpanel);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(aux->join[0], aux->st[0])) != cudaSuccess) return e;
  k3_stage_a<<<dim3(blocks(amax), ng), 256, 0, s>>>(p->d_groups, rowperm, p->d_perm[1], gk, p->chi[1],
                                                     lk, p->d_apanel);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaStreamWaitEvent(s, aux->join[0], 0);
}

}  // namespace tn
