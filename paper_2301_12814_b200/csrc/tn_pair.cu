// MPO (doubled-charge) plans — Θ(c1, c2) of PAPER.md:101, :107 ("MPOs are vectorized into the MPS form,
// U → U⊗U*, and two conserved charges are present"). DESIGN.md §4 "Pair plans".
//
// A bond carries a charge pair (c1, c2); K1 sorts bonds by the lexicographic key c1·(N+1) + c2,
// so every charge PAIR is one contiguous segment of sorted positions. The product-once reformulation of
// the single-charge path carries over pair by pair:
//   P_m = A_m · B_m for every centre pair m = (m1, m2)   (K3 staging + K4 contraction, unchanged kernels)
//   Θ(c1,c2)[α,β] = λlλr Σ_{m1,m2} U_{n1}[l1−c1][l1−m1] · conj(U_{n2}[l2−c2][l2−m2]) · P_m[α,β]
// and the U⊗U* weight factorises, so the mix is applied one species at a time (K5P, two passes):
//   pass 1:  Q(c1, m2) = Σ_{m1} U_{n1}[l1−c1][l1−m1] P(m1, m2)              (in place, per m2)
//   pass 2:  Θ(c1, c2) = λlλr Σ_{m2} conj(U_{n2}[l2−c2][l2−m2]) Q(c1, m2)     (in place, per c1)
// L1²L2 + L1L2² complex MACs per element instead of (L1L2)². Blocks whose two vectors are short (L1, L2 ≤ 8) take
// both factors in ONE pass instead (K5F: Y = U1·X·U2ᴴ per element in shared memory / registers), reading and
// writing Θ once. Sector (c1, c2) is compact row-major; its rows
// are the sorted left positions with l − c ∈ [0, d−1]² — a union of whole pair segments, in sorted order —
// and its columns likewise. P_m has exactly Θ(m)'s shape, so K4 writes it straight into Θ(m) as before;
// the group's rows/columns are gathered through per-group position lists (d_rowperm / d_colperm).
#include <chrono>
#include <numeric>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "k5_mix.cuh"

namespace tn {

__global__ void k_gather_idx(int32_t* __restrict__ out, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ pos, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = perm[pos[i]];
}

namespace {
struct Carve {  // bump allocator over one pool block (256-byte aligned pieces)
  size_t off = 0;
  template <class T>
  size_t take(int64_t n) {
    const size_t o = off;
    off += ((size_t)std::max<int64_t>(n, 0) * sizeof(T) + 255) & ~(size_t)255;
    return o;
  }
};
}  // namespace

tn_status build_pair_tables(tn_plan* p) {
  // TN_PLAN_PROFILE=1: host µs per phase on stderr
  static const bool prof = getenv("TN_PLAN_PROFILE") != nullptr;
  double pt[10] = {};
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
#define PP(i) \
  if (prof) pt[i] = now_us()
  PP(0);
  const int N = p->N, d = p->d, nk = N + 1, nq = p->nq;
  const auto& ol = p->off[0];
  const auto& oc = p->off[1];
  const auto& orr = p->off[2];
  auto cnt = [](const std::vector<int32_t>& o, int k) { return (int64_t)o[k + 1] - o[k]; };
  // For a (left pair l, right pair r) block the admissible centre pairs are the rectangle I1 × I2, Ik = [max(rk,
  // lk−d+1), min(lk, rk+d−1)] (both species' δ's): their count L1·L2 and Σ n_c over it come from a 2-D prefix
  // sum over the centre-pair counts, O(1) per block instead of a scan over all (N+1)² centre pairs.
  std::vector<int64_t> P2((size_t)(nk + 1) * (nk + 1), 0);   // P2[(a)(nk+1) + b] = Σ_{m1<a, m2<b} n_c(m1, m2)
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nk; ++b)
      P2[(size_t)(a + 1) * (nk + 1) + b + 1] = P2[(size_t)a * (nk + 1) + b + 1] + P2[(size_t)(a + 1) * (nk + 1) + b] -
                                               P2[(size_t)a * (nk + 1) + b] + cnt(oc, a * nk + b);
  // the non-empty left / right pair keys with their charges: the O(keys²) loops below visit only these (no
  // divisions by N+1 in them)
  struct Key {
    int k, k1, k2;
    int64_t n;
  };
  std::vector<Key> lkeys, rkeys;
  for (int k = 0; k < nq; ++k) {
    if (cnt(ol, k)) lkeys.push_back(Key{k, k / nk, k % nk, cnt(ol, k)});
    if (cnt(orr, k)) rkeys.push_back(Key{k, k / nk, k % nk, cnt(orr, k)});
  }
  PP(1);
  // ---- sector layouts: local row / column offset of every pair segment inside every sector ----
  std::vector<int32_t>& rowoff = p->h_rowoff;
  std::vector<int32_t>& coloff = p->h_coloff;
  rowoff.assign((size_t)nq * nq, -1);
  coloff.assign((size_t)nq * nq, -1);
  p->R.assign(nq, 0);
  p->C.assign(nq, 0);
  p->row0.assign(nq, 0);
  p->col0.assign(nq, 0);
  p->lR.assign(nq, 0);
  p->lrow0.assign(nq, 0);
  PP(2);
  // ---- flop-balanced row shards over sorted left positions (per-pair row cost: contraction + mix) ----
  // per left key: Σ_r n_r·(centre count) and Σ_r n_r·(mix MACs) — the row cost, and (× rows) the flop counts below
  std::vector<int64_t> lmc(nq, 0), lmx(nq, 0);
  {
    std::vector<double> cost(nq, 0.0);
    for (const Key& L : lkeys) {
      int64_t smc = 0, smx = 0;
      for (const Key& R : rkeys) {
        const int a0 = std::max(R.k1, L.k1 - d + 1), a1 = std::min(L.k1, R.k1 + d - 1);
        const int b0 = std::max(R.k2, L.k2 - d + 1), b1 = std::min(L.k2, R.k2 + d - 1);
        if (a1 < a0 || b1 < b0) continue;
        const int64_t L1 = a1 - a0 + 1, L2 = b1 - b0 + 1;
        const int64_t mc = P2[(size_t)(a1 + 1) * (nk + 1) + b1 + 1] - P2[(size_t)a0 * (nk + 1) + b1 + 1] -
                           P2[(size_t)(a1 + 1) * (nk + 1) + b0] + P2[(size_t)a0 * (nk + 1) + b0];
        smc += R.n * mc;
        smx += R.n * (L1 * L1 * L2 + L1 * L2 * L2);
      }
      lmc[L.k] = smc;
      lmx[L.k] = smx;
      cost[L.k] = (double)smc + (double)smx;
    }
    double total = 0.0;
    for (int l = 0; l < nq; ++l) total += cost[l] * (double)cnt(ol, l);
    const int W = p->world;
    p->bounds.assign(W + 1, 0);
    p->bounds[W] = p->chi[0];
    double prefix = 0.0;
    int64_t row = 0;
    int rk = 1;
    for (int l = 0; l < nq && rk < W; ++l)
      for (int64_t i = 0; i < cnt(ol, l) && rk < W; ++i) {
        while (rk < W && prefix >= total * (double)rk / W) p->bounds[rk++] = row;
        prefix += cost[l];
        ++row;
      }
    while (rk < W) p->bounds[rk++] = row;
    p->r0 = p->bounds[p->rank];
    p->r1 = p->bounds[p->rank + 1];
  }
  const int64_t R0 = p->r0, R1 = p->r1;
  auto in_shard = [&](int l) {  // rows of left segment l inside [r0, r1): [first, count)
    const int64_t a = std::max<int64_t>(ol[l], R0), b = std::min<int64_t>(ol[l + 1], R1);
    return std::make_pair(a, std::max<int64_t>(0, b - a));
  };
  for (int c1 = 0; c1 <= N; ++c1)
    for (int c2 = 0; c2 <= N; ++c2) {
      const int s = c1 * nk + c2;
      // rows of Θ(s): whole left segments in key (= sorted) order; this rank's slab = those in [r0, r1),
      // one contiguous run of Θ(s)'s rows starting at a_s = #rows of Θ(s) before r0
      int64_t r = 0, c = 0, a_s = 0, rl = 0;
      for (int l1 = c1; l1 <= std::min(N, c1 + d - 1); ++l1)
        for (int l2 = c2; l2 <= std::min(N, c2 + d - 1); ++l2) {
          const int l = l1 * nk + l2;
          a_s += std::min<int64_t>(std::max<int64_t>(R0 - ol[l], 0), cnt(ol, l));
          rl += in_shard(l).second;
        }
      for (int l1 = c1; l1 <= std::min(N, c1 + d - 1); ++l1)
        for (int l2 = c2; l2 <= std::min(N, c2 + d - 1); ++l2) {
          const int l = l1 * nk + l2;
          // slab-local row of segment l's first in-shard row
          rowoff[(size_t)s * nq + l] =
              (int32_t)(r + std::min<int64_t>(std::max<int64_t>(R0 - ol[l], 0), cnt(ol, l)) - a_s);
          r += cnt(ol, l);
        }
      for (int r1 = std::max(0, c1 - d + 1); r1 <= c1; ++r1)
        for (int r2 = std::max(0, c2 - d + 1); r2 <= c2; ++r2) {
          coloff[(size_t)s * nq + r1 * nk + r2] = (int32_t)c;
          c += cnt(orr, r1 * nk + r2);
        }
      if (r > INT32_MAX || c > INT32_MAX) return fail(TN_ERR_UNSUPPORTED, "sector dimension > INT32_MAX");
      p->R[s] = r;
      p->lR[s] = rl;
      p->lrow0[s] = rl ? a_s : 0;  // pair plans: slab start as a row index of Θ(s) (row0 = 0)
      p->C[s] = c;
    }
  PP(3);
  // ---- useful work (oracle.flop_counts2 definitions), from the per-left-key sums above ----
  p->f_contract = p->f_mix = 0;
  p->f_contract_local = p->f_mix_local = 0;
  for (const Key& L : lkeys) {
    const int64_t nll = in_shard(L.k).second;
    p->f_contract += 8 * L.n * lmc[L.k];
    p->f_mix += 8 * L.n * lmx[L.k];
    p->f_contract_local += 8 * nll * lmc[L.k];
    p->f_mix_local += 8 * nll * lmx[L.k];
  }
  PP(4);
  // ---- groups: one per non-empty centre pair; rows / cols = those of Θ(m), gathered by position ----
  std::vector<int32_t>& rpos = p->h_rowperm_pos;
  std::vector<int32_t>& cpos = p->h_colperm_pos;
  rpos.clear();
  cpos.clear();
  int64_t a_off = 0, b_off = 0;
  p->groups.clear();
  p->f_exec = 0;
  for (int m = 0; m < nq; ++m) {
    const int64_t K = cnt(oc, m);
    if (K == 0 || p->lR[m] == 0 || p->C[m] == 0) continue;
    const int m1 = m / nk, m2 = m % nk;
    GroupDesc g{};
    g.cc = m;
    g.row0 = (int64_t)rpos.size();
    rpos.resize(rpos.size() + (size_t)p->lR[m]);   // whole runs of consecutive positions: fill, no push_back
    {
      int32_t* w = rpos.data() + g.row0;
      for (int l1 = m1; l1 <= std::min(N, m1 + d - 1); ++l1)
        for (int l2 = m2; l2 <= std::min(N, m2 + d - 1); ++l2) {
          const auto sh = in_shard(l1 * nk + l2);
          std::iota(w, w + sh.second, (int32_t)sh.first);
          w += sh.second;
        }
    }
    g.col0 = (int64_t)cpos.size();
    cpos.resize(cpos.size() + (size_t)p->C[m]);
    {
      int32_t* w = cpos.data() + g.col0;
      for (int r1 = std::max(0, m1 - d + 1); r1 <= m1; ++r1)
        for (int r2 = std::max(0, m2 - d + 1); r2 <= m2; ++r2) {
          const int rk = r1 * nk + r2;
          std::iota(w, w + cnt(orr, rk), orr[rk]);
          w += cnt(orr, rk);
        }
    }
    g.k0 = oc[m];
    g.R = (int32_t)p->lR[m];
    g.C = (int32_t)p->C[m];
    g.K = (int32_t)K;
    g.K4 = (int32_t)((K + 3) / 4 * 4);
    g.nmt = (g.R + BM - 1) / BM;
    g.nnt = (g.C + BN - 1) / BN;
    g.a_off = a_off;
    g.b_off = b_off;
    a_off += (int64_t)g.nmt * BM * g.K4;
    b_off += (int64_t)g.nnt * BN * g.K4;
    p->f_exec += 8 * (int64_t)g.nmt * BM * (int64_t)g.nnt * BN * g.K4;
    p->groups.push_back(g);
  }
  p->a_elems = a_off;
  p->b_elems = b_off;
  std::vector<int> order(p->groups.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p->groups[x].K4 > p->groups[y].K4; });
  std::vector<TileDesc>& tiles = p->h_tiles;
  tiles.clear();
  for (int gi : order)
    for (int mt = 0; mt < p->groups[gi].nmt; ++mt)
      for (int nt = 0; nt < p->groups[gi].nnt; ++nt) tiles.push_back(TileDesc{gi, mt, nt, 0});
  p->ntiles = (int64_t)tiles.size();
  PP(5);
  // ---- two-pass mix tiles: rows of one left pair segment (≈ 128 8-groups) × one right pair segment ----
  // Within a pass: single-value tiles first, then the multi-value ones (launched with the MULTI kernel, whose
  // extra index arithmetic the common single-value tiles do not pay); inside each, by register class of L (one
  // launch per class: a kernel sized for the largest L of the plan held every tile at its register count — the
  // K5 register classes of the single-charge path). Two walks — count per bucket, then write each
  // tile straight into its bucket — keep this loop (≈ 10⁵ tiles at pair config 5, on the per-gate plan's path)
  // free of reallocation, sorting and copies.
  std::vector<MixTile2>& mix = p->h_mix2;
  mix.clear();
  p->nfix_max = 1;
  int max_l = 1;
  auto cls = [](int L) { return L <= 8 ? 0 : L <= 16 ? 1 : L <= 32 ? 2 : 3; };
  // Blocks whose both species' vectors are short (L1, L2 ≤ 8) are mixed by K5F in one pass (Θ read and written once);
  // longer ones keep the two passes, which run on the tensor pipe (measured: K5F with L up to 18 held one CTA per
  // SM at 130–200 registers and lost to the two passes: pair config 5 4.68 vs 3.18 ms; at L ≤ 8 it wins, pair
  // config 3 0.51 vs 0.80 ms). TN_PAIR_TWO_PASS=1 sends every block through the two passes.
  const bool two_pass = getenv("TN_PAIR_TWO_PASS") != nullptr;   // read per plan (tests switch it)
  constexpr int FUSE_MAXL = 8;
  // One enumeration of the (left key, right key) blocks of this shard computes every block's tile counts per launch
  // bucket (a tile of a block has the block's L; only its last value group may cover fewer values of the other
  // species); a prefix over the blocks gives each block's first slot per bucket, and one fill loop writes every
  // tile straight into place — no sorting, copies or per-tile reallocation on the per-gate plan's path.
  // Buckets: 0 = K5F; 1 + pass·8 + (multi ? 4 : 0) + class(L) for the two-pass tiles (single-value first).
  constexpr int NB = 17;
  struct BlkT {
    int li, ri, lo1, hi1, lo2, hi2;
    int64_t nl, lfirst, ngr, rows_per;
    int nfix[2];      // 0, 0: a K5F block
  };
  std::vector<BlkT> blocks;
  blocks.reserve(lkeys.size() * rkeys.size());
  int64_t tot[NB] = {};
  for (int li = 0; li < (int)lkeys.size(); ++li) {
    const Key& Lk = lkeys[li];
    const auto sh = in_shard(Lk.k);
    if (!sh.second) continue;
    for (int ri = 0; ri < (int)rkeys.size(); ++ri) {
      const Key& Rk = rkeys[ri];
      BlkT b;
      b.lo1 = std::max(Rk.k1, Lk.k1 - d + 1);
      b.hi1 = std::min(Lk.k1, Rk.k1 + d - 1);
      b.lo2 = std::max(Rk.k2, Lk.k2 - d + 1);
      b.hi2 = std::min(Lk.k2, Rk.k2 + d - 1);
      if (b.hi1 < b.lo1 || b.hi2 < b.lo2) continue;
      b.li = li;
      b.ri = ri;
      b.nl = sh.second;
      b.lfirst = sh.first;
      b.ngr = (Rk.n + 7) / 8;
      b.rows_per = std::max<int64_t>(1, MIX_GROUPS_PER_TILE / b.ngr);
      const int L1 = b.hi1 - b.lo1 + 1, L2 = b.hi2 - b.lo2 + 1;
      const int64_t bands = (b.nl + b.rows_per - 1) / b.rows_per;
      max_l = std::max(max_l, std::max(L1, L2));
      if (!two_pass && L1 <= FUSE_MAXL && L2 <= FUSE_MAXL) {
        tot[0] += bands;
        b.nfix[0] = b.nfix[1] = 0;
      } else {
        for (int pass = 0; pass < 2; ++pass) {
          const int L = pass == 0 ? L1 : L2, span = pass == 0 ? L2 : L1;
          // several values of the other species per tile when one value's band is small (≈ 128 8-groups a tile)
          const int64_t per_val = std::min<int64_t>(b.rows_per, b.nl) * b.ngr;
          const int nfix = (int)std::max<int64_t>(1, std::min<int64_t>(span, MIX_GROUPS_PER_TILE / std::max<int64_t>(1, per_val)));
          b.nfix[pass] = nfix;
          p->nfix_max = std::max(p->nfix_max, nfix);
          const int ngrp = (span + nfix - 1) / nfix, nf_last = span - (ngrp - 1) * nfix;
          tot[1 + pass * 8 + (nfix == 1 ? 0 : 4) + cls(L)] += (ngrp - 1) * bands;
          tot[1 + pass * 8 + (nf_last == 1 ? 0 : 4) + cls(L)] += bands;
        }
      }
      blocks.push_back(b);
    }
  }
  int64_t at[NB], all = 0;
  for (int g = 0; g < NB; ++g) {
    at[g] = all;
    all += tot[g];
  }
  mix.resize((size_t)all);
  MixTile2* o = mix.data();
  for (const BlkT& b : blocks) {
    const Key& Lk = lkeys[b.li];
    const Key& Rk = rkeys[b.ri];
    const int L1 = b.hi1 - b.lo1 + 1, L2 = b.hi2 - b.lo2 + 1;
    auto base_tile = [&](int64_t band) {
      MixTile2 t{};
      t.e0 = 0;
      t.ne = (int32_t)(std::min<int64_t>(b.rows_per, b.nl - band) * b.ngr);
      t.nr = (int32_t)Rk.n;
      t.ngr = (int32_t)b.ngr;
      t.pl0 = (int32_t)(b.lfirst + band);
      t.pr0 = orr[Rk.k];
      t.lkey = Lk.k;
      t.rkey = Rk.k;
      t.band = (int32_t)band;
      return t;
    };
    if (b.nfix[0] == 0) {   // K5F: species 1 in (cl, n, lo, L), species 2's lo / L in fixed / nfix
      for (int64_t band = 0; band < b.nl; band += b.rows_per) {
        MixTile2 t = base_tile(band);
        t.cl = Lk.k1;
        t.n = Lk.k1 - Rk.k1;
        t.lo = b.lo1;
        t.L = L1;
        t.fixed = b.lo2;
        t.nfix = L2;
        t.flags = 2;
        o[at[0]++] = t;
      }
      continue;
    }
    for (int pass = 0; pass < 2; ++pass) {
      const int L = pass == 0 ? L1 : L2;
      const int fixed_lo = pass == 0 ? b.lo2 : b.lo1, fixed_hi = pass == 0 ? b.hi2 : b.hi1, nfix = b.nfix[pass];
      for (int f = fixed_lo; f <= fixed_hi; f += nfix) {
        const int nf = std::min(nfix, fixed_hi - f + 1);
        const int g = 1 + pass * 8 + (nf == 1 ? 0 : 4) + cls(L);
        for (int64_t band = 0; band < b.nl; band += b.rows_per) {
          MixTile2 t = base_tile(band);
          t.cl = pass == 0 ? Lk.k1 : Lk.k2;
          t.n = pass == 0 ? Lk.k1 - Rk.k1 : Lk.k2 - Rk.k2;
          t.lo = pass == 0 ? b.lo1 : b.lo2;
          t.L = L;
          t.fixed = f;
          t.nfix = nf;
          t.flags = pass;
          o[at[g]++] = t;
        }
      }
    }
  }
  p->nmix_fused = tot[0];
  for (int pass = 0; pass < 2; ++pass) {
    int64_t n = 0;
    for (int m = 0; m < 2; ++m)
      for (int c = 0; c < 4; ++c) {
        p->nmix2_grp[pass][m][c] = tot[1 + pass * 8 + m * 4 + c];
        n += p->nmix2_grp[pass][m][c];
      }
    p->nmix2[pass] = n;
    p->nmix2_multi[pass] = n - (p->nmix2_grp[pass][0][0] + p->nmix2_grp[pass][0][1] + p->nmix2_grp[pass][0][2] +
                                p->nmix2_grp[pass][0][3]);
  }
  p->max_mix = max_l;
  p->nmix = 0;
  PP(6);
  // ---- device tables ----
  Carve cw;
  const size_t o_g = cw.take<GroupDesc>((int64_t)p->groups.size());
  const size_t o_t = cw.take<TileDesc>((int64_t)tiles.size());
  const size_t o_m = cw.take<MixTile2>((int64_t)mix.size());
  const size_t o_ro = cw.take<int32_t>((int64_t)nq * nq);
  const size_t o_co = cw.take<int32_t>((int64_t)nq * nq);
  const size_t o_rp = cw.take<int32_t>((int64_t)rpos.size());
  const size_t o_cp = cw.take<int32_t>((int64_t)cpos.size());
  const size_t o_rg = cw.take<int32_t>((int64_t)rpos.size());
  const size_t o_cg = cw.take<int32_t>((int64_t)cpos.size());
  const size_t o_a = cw.take<double2>(p->a_elems);
  const size_t o_b = cw.take<double2>(p->b_elems);
  cudaError_t aerr = cudaSuccess;
  p->blk_work = pool_alloc(cw.off, &aerr);
  if (aerr != cudaSuccess) return cuda_check(aerr, "pool alloc (pair workspace)");
  char* base = static_cast<char*>(p->blk_work);
  p->d_groups = reinterpret_cast<GroupDesc*>(base + o_g);
  p->d_tiles = reinterpret_cast<TileDesc*>(base + o_t);
  p->d_mix2 = reinterpret_cast<MixTile2*>(base + o_m);
  p->d_rowoff = reinterpret_cast<int32_t*>(base + o_ro);
  p->d_coloff = reinterpret_cast<int32_t*>(base + o_co);
  int32_t* d_rpos = reinterpret_cast<int32_t*>(base + o_rp);
  int32_t* d_cpos = reinterpret_cast<int32_t*>(base + o_cp);
  int32_t* d_rg = reinterpret_cast<int32_t*>(base + o_rg);
  int32_t* d_cg = reinterpret_cast<int32_t*>(base + o_cg);
  p->d_apanel = reinterpret_cast<double2*>(base + o_a);
  p->d_bpanel = reinterpret_cast<double2*>(base + o_b);
  p->d_rowperm = d_rg;
  p->d_colperm = d_cg;
  p->d_rowpos = d_rpos;
  p->n_rowlist = (int64_t)rpos.size();
  p->ws_bytes += (int64_t)cw.off;
  auto up = [&](void* dst, const void* src, size_t bytes, const char* what) -> tn_status {
    if (!bytes) return TN_OK;
    return cuda_check(plan_h2d(p, dst, src, bytes), what);
  };
  tn_status st;
  if ((st = up(p->d_groups, p->groups.data(), p->groups.size() * sizeof(GroupDesc), "H2D groups")) != TN_OK) return st;
  if ((st = up(p->d_tiles, tiles.data(), tiles.size() * sizeof(TileDesc), "H2D tiles")) != TN_OK) return st;
  if ((st = up(p->d_mix2, mix.data(), mix.size() * sizeof(MixTile2), "H2D mix tiles")) != TN_OK) return st;
  if ((st = up(p->d_rowoff, rowoff.data(), rowoff.size() * sizeof(int32_t), "H2D row offsets")) != TN_OK) return st;
  if ((st = up(p->d_coloff, coloff.data(), coloff.size() * sizeof(int32_t), "H2D col offsets")) != TN_OK) return st;
  if ((st = up(d_rpos, rpos.data(), rpos.size() * sizeof(int32_t), "H2D row positions")) != TN_OK) return st;
  if ((st = up(d_cpos, cpos.data(), cpos.size() * sizeof(int32_t), "H2D col positions")) != TN_OK) return st;
  // gathered index lists: original bond index of every group row / column (K1's perm already on device)
  if (!rpos.empty())
    k_gather_idx<<<(unsigned)std::min<int64_t>(1024, ((int64_t)rpos.size() + 255) / 256), 256, 0, p->plan_stream>>>(
        d_rg, p->d_perm[0], d_rpos, (int64_t)rpos.size());
  if (!cpos.empty())
    k_gather_idx<<<(unsigned)std::min<int64_t>(1024, ((int64_t)cpos.size() + 255) / 256), 256, 0, p->plan_stream>>>(
        d_cg, p->d_perm[2], d_cpos, (int64_t)cpos.size());
  PP(7);
  if (prof)
    fprintf(stderr, "[plan2] us: P2 %.1f layouts %.1f shards %.1f flops %.1f groups+tiles %.1f mix %.1f (%zu tiles) "
            "tables+uploads %.1f\n", pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[5] - pt[4],
            pt[6] - pt[5], p->h_mix2.size(), pt[7] - pt[6]);
#undef PP
  return cuda_check(cudaGetLastError(), "pair gather launch");
}

// ---- K5P: one species' mix of one pair tile (same warp loop as K5, sector list from the plan) ----
constexpr int K5P_THREADS = 128;

template <int NTMAX, bool MULTI>
__global__ void __launch_bounds__(K5P_THREADS, (NTMAX == 1 ? 8 : NTMAX == 2 ? 7 : NTMAX <= 4 ? 4 : 2))
    k5p_mix(const SectorParams sp, const MixTile2* __restrict__ tiles, const int32_t* __restrict__ rowoff,
            const int32_t* __restrict__ coloff, int nq, const int32_t* __restrict__ perm_l,
            const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
            const double2* __restrict__ U, int us_elems, int nfix_max) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const MixTile2 t = tiles[blockIdx.x];
  // nfix_max sector tables (one per value of the other species the tile covers), each 8·NTMAX entries
  constexpr int SSTR = 8 * NTMAX;
  SecRef* ld_sec = reinterpret_cast<SecRef*>(smem_raw);
  SecRef* st_sec = ld_sec + SSTR * nfix_max;
  double2* Us = reinterpret_cast<double2*>(st_sec + SSTR * nfix_max);
  double* UsS = reinterpret_cast<double*>(Us + us_elems);
  const int L = t.L, d = sp.d, nk = sp.N + 1;
  const bool pass2 = t.flags & 1;
  // the sector tables of the tile's nfix values f of the other species: pass 1 sectors (lo+u, f), sources valid
  // only for a non-empty centre pair; pass 2 sectors (f, lo+u)
  const int nfix = MULTI ? t.nfix : 1;
  for (int x = threadIdx.x; x < L * nfix; x += K5P_THREADS) {
    const int fi = x / L, u = x - fi * L, f = t.fixed + fi;
    const int s = pass2 ? f * nk + t.lo + u : (t.lo + u) * nk + f;
    const SecEntry e = sp.sec[s];
    const int64_t off = (int64_t)(rowoff[s * nq + t.lkey] + t.band) * e.ld + coloff[s * nq + t.rkey];
    const double2* base = e.out + off;
    const bool valid = pass2 || e.nonempty;
    // the source is Θ(s) itself, or a local workspace when Θ goes elsewhere (tn_theta_exec_remote, pass 2)
    const double2* lbase = e.src ? e.src + off : base;
    ld_sec[fi * SSTR + u] = SecRef{valid ? lbase : nullptr, (int64_t)e.ld};
    st_sec[fi * SSTR + u] = SecRef{base, (int64_t)e.ld};
  }
  // Us[t][u] = U_n[i = cl − (lo+t)][j = cl − (lo+u)]  (conjugated for the bra species), padded to TP × UP
  const int TP = (L + 7) & ~7, UP = (L + 3) & ~3;
  const int ust = us_stride(UP);
  const int nlo = max(0, t.n - d + 1), sn = min(t.n, d - 1) - nlo + 1;
  const double2* Ub = U + sp.ustart[t.n];
  for (int x = threadIdx.x; x < TP * UP; x += K5P_THREADS) {
    const int tt = x / UP, u = x - tt * UP;
    double2 v = make_double2(0.0, 0.0);
    if (tt < L && u < L) {
      v = __ldg(Ub + (t.cl - t.lo - tt - nlo) * sn + (t.cl - t.lo - u - nlo));
      if (pass2) v.y = -v.y;  // the bra species carries conj(U)
    }
    Us[tt * ust + u] = v;
    UsS[tt * ust + u] = v.x + v.y;
  }
  __syncthreads();
  MixTile mt;
  mt.cl = t.cl;
  mt.cr = 0;
  mt.e0 = t.e0;
  mt.ne = t.ne;
  mt.nr = t.nr;
  mt.ngr = t.ngr;
  mt.pl0 = t.pl0;
  mt.pr0 = t.pr0;
  const bool sc = pass2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the tile's nfix values form one 8-group index space (several small pair segments per CTA)
  switch (TP >> 3) {
#define TN_MIX_CASE(m)                                                                                       \
  case m:                                                                                                    \
    if constexpr (m <= NTMAX)                                                                                \
      mix_tile_warp<m, K5P_THREADS / 32, false, 0, MULTI>(mt, ld_sec, st_sec, Us, UsS, ust, L, perm_l, perm_r, \
                                                          sc ? ll : nullptr, lr, warp, lane, nfix, SSTR);    \
    break;
    TN_MIX_CASE(1) TN_MIX_CASE(2) TN_MIX_CASE(3) TN_MIX_CASE(4)
    TN_MIX_CASE(5) TN_MIX_CASE(6) TN_MIX_CASE(7) TN_MIX_CASE(8)
#undef TN_MIX_CASE
    default:
      break;
  }
}

// ---- K5F: both species' mix of one pair tile in ONE pass (DESIGN.md §4 "Pair plans") ----
// For every element (α, β) of the tile's (l, r) block the L1 × L2 values X[i][j] = P(lo1+i, lo2+j)[α, β] become
// Θ(lo1+t, lo2+u)[α, β] = λlλr Σ_{i,j} U_{n1}[l1−lo1−t][l1−lo1−i] · conj(U_{n2}[l2−lo2−u][l2−lo2−j]) · X[i][j], i.e.
// Y = U1·X·U2ᴴ: the CTA stages a chunk of E elements' X blocks in shared memory (coalesced 128-byte runs per
// sector), applies U1 down the columns (one thread per (j, e), L1 values in registers) and U2* along the rows (one
// thread per (t, e)), and stores Y straight from registers. Θ is read once and written once — the two-pass K5P
// moved it twice (pass 1 and pass 2 each read and wrote every element).
constexpr int K5F_THREADS = 256;
constexpr int K5F_X_BYTES = 64 * 1024;   // X chunk budget (E = 8·G elements per chunk, G 8-groups; two CTAs per SM)

template <int LMAX>
__global__ void __launch_bounds__(K5F_THREADS, 2)
    k5f_mix(const SectorParams sp_ld, const SectorParams sp_st, const MixTile2* __restrict__ tiles,
            const int32_t* __restrict__ rowoff, const int32_t* __restrict__ coloff, int nq,
            const int32_t* __restrict__ perm_l, const int32_t* __restrict__ perm_r, const double* __restrict__ ll,
            const double* __restrict__ lr, const double2* __restrict__ U) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double2* U1s = reinterpret_cast<double2*>(smem_raw);                 // [LMAX][LMAX]
  double2* U2s = U1s + LMAX * LMAX;                                    // conj, [u][j]
  uint8_t* tab = reinterpret_cast<uint8_t*>(U2s + LMAX * LMAX);
  const double2** ldp = reinterpret_cast<const double2**>(tab);                          // [L1·L2] load base (nullptr: P = 0)
  double2** stp = reinterpret_cast<double2**>(tab + LMAX * LMAX * sizeof(void*));         // [L1·L2] store base
  int64_t* ldv = reinterpret_cast<int64_t*>(tab + 2 * LMAX * LMAX * sizeof(void*));      // [L1·L2] load row stride
  int64_t* stv = ldv + LMAX * LMAX;                                              // [L1·L2] store row stride
  double2* X = reinterpret_cast<double2*>(stv + LMAX * LMAX);                    // [L1·L2][E]
  const MixTile2 t = tiles[blockIdx.x];
  const int nk = sp_ld.N + 1, d = sp_ld.d;
  const int L1 = t.L, lo1 = t.lo, L2 = t.nfix, lo2 = t.fixed;
  const int l1 = t.cl, n1 = t.n, l2 = t.lkey % nk, n2 = l2 - t.rkey % nk;
  const int LL = L1 * L2;
  const int tid = threadIdx.x;
  for (int x = tid; x < LL; x += K5F_THREADS) {
    const int i = x / L2, j = x - i * L2;
    const int s = (lo1 + i) * nk + lo2 + j;
    const SecEntry el = sp_ld.sec[s], es = sp_st.sec[s];
    const int64_t off = (int64_t)(rowoff[s * nq + t.lkey] + t.band) * el.ld + coloff[s * nq + t.rkey];
    ldp[x] = el.nonempty ? (el.src ? el.src : el.out) + off : nullptr;
    stp[x] = es.out + ((int64_t)(rowoff[s * nq + t.lkey] + t.band) * es.ld + coloff[s * nq + t.rkey]);
    ldv[x] = el.ld;
    stv[x] = es.ld;
  }
  {
    const int nlo1 = max(0, n1 - d + 1), sn1 = min(n1, d - 1) - nlo1 + 1;
    const int nlo2 = max(0, n2 - d + 1), sn2 = min(n2, d - 1) - nlo2 + 1;
    const double2* Ub1 = U + sp_ld.ustart[n1];
    const double2* Ub2 = U + sp_ld.ustart[n2];
    for (int x = tid; x < L1 * L1; x += K5F_THREADS) {
      const int a = x / L1, b = x - a * L1;
      U1s[a * LMAX + b] = __ldg(Ub1 + (l1 - lo1 - a - nlo1) * sn1 + (l1 - lo1 - b - nlo1));
    }
    for (int x = tid; x < L2 * L2; x += K5F_THREADS) {
      const int a = x / L2, b = x - a * L2;
      const double2 v = __ldg(Ub2 + (l2 - lo2 - a - nlo2) * sn2 + (l2 - lo2 - b - nlo2));
      U2s[a * LMAX + b] = make_double2(v.x, -v.y);   // the bra species carries conj(U)
    }
  }
  __syncthreads();
  const int G = max(1, K5F_X_BYTES / (LL * 8 * (int)sizeof(double2)));   // 8-groups per chunk
  for (int k0 = 0; k0 < t.ne; k0 += G) {
    const int ng = min(G, t.ne - k0), E = 8 * ng;
    // stage X[ij][e]: consecutive threads → consecutive columns of one sector row (128-byte runs); 8 loads in
    // flight per thread before any is stored (one at a time left every warp waiting out a full HBM latency per load)
    constexpr int MLP = 8;
    for (int x0 = tid; x0 < LL * E; x0 += K5F_THREADS * MLP) {
      double2 v[MLP];
#pragma unroll
      for (int q = 0; q < MLP; ++q) {
        const int x = x0 + q * K5F_THREADS;
        v[q] = make_double2(0.0, 0.0);
        if (x < LL * E) {
          const int ij = x / E, e = x - ij * E;
          const int grp = t.e0 + k0 + (e >> 3);
          const int row = grp / t.ngr, col = (grp - row * t.ngr) * 8 + (e & 7);
          const double2* b = ldp[ij];
          if (b && col < t.nr) v[q] = __ldcg(b + (int64_t)row * ldv[ij] + col);
        }
      }
#pragma unroll
      for (int q = 0; q < MLP; ++q) {
        const int x = x0 + q * K5F_THREADS;
        if (x < LL * E) X[x] = v[q];
      }
    }
    __syncthreads();
    // U1 down every column (j, e): X[:, j, e] ← U1 · X[:, j, e] — the column's L1 inputs and all L1 outputs in
    // registers, input-major, so the L1 output accumulations are independent (no dependent FMA chains)
    for (int y = tid; y < L2 * E; y += K5F_THREADS) {
      const int j = y / E, e = y - j * E;
      double2 acc[LMAX];
#pragma unroll
      for (int a = 0; a < LMAX; ++a) acc[a] = make_double2(0.0, 0.0);
      for (int i = 0; i < L1; ++i) {
        const double2 v = X[(i * L2 + j) * E + e];
#pragma unroll
        for (int a = 0; a < LMAX; ++a)
          if (a < L1) {
            const double2 u = U1s[a * LMAX + i];
            acc[a].x = fma(u.x, v.x, fma(-u.y, v.y, acc[a].x));
            acc[a].y = fma(u.x, v.y, fma(u.y, v.x, acc[a].y));
          }
      }
#pragma unroll
      for (int a = 0; a < LMAX; ++a)
        if (a < L1) X[(a * L2 + j) * E + e] = acc[a];
    }
    __syncthreads();
    // U2* along every row (a, e), λlλr, store: Θ(lo1+a, lo2+u)[row, col]
    for (int y = tid; y < L1 * E; y += K5F_THREADS) {
      const int a = y / E, e = y - a * E;
      const int grp = t.e0 + k0 + (e >> 3);
      const int row = grp / t.ngr, col = (grp - row * t.ngr) * 8 + (e & 7);
      if (col >= t.nr) continue;
      double2 acc[LMAX];
#pragma unroll
      for (int u = 0; u < LMAX; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int j = 0; j < L2; ++j) {
        const double2 v = X[(a * L2 + j) * E + e];
#pragma unroll
        for (int u = 0; u < LMAX; ++u)
          if (u < L2) {
            const double2 w = U2s[u * LMAX + j];
            acc[u].x = fma(w.x, v.x, fma(-w.y, v.y, acc[u].x));
            acc[u].y = fma(w.x, v.y, fma(w.y, v.x, acc[u].y));
          }
      }
      const double scale = ll ? ll[perm_l[t.pl0 + row]] * lr[perm_r[t.pr0 + col]] : 1.0;
#pragma unroll
      for (int u = 0; u < LMAX; ++u)
        if (u < L2) {
          const int ij = a * L2 + u;
          __stcg(stp[ij] + (int64_t)row * stv[ij] + col, make_double2(acc[u].x * scale, acc[u].y * scale));
        }
    }
    __syncthreads();
  }
}

static cudaError_t launch_pair_mix_fused(const tn_plan* p, const SectorParams& sp_ld, const SectorParams& sp_st,
                                         const double* ll, const double* lr, const double2* U, cudaStream_t s) {
  if (p->nmix_fused == 0) return cudaSuccess;
  constexpr int LM = 8;
  const size_t smem = (size_t)2 * LM * LM * sizeof(double2) + (size_t)LM * LM * (2 * sizeof(void*) + 16) + K5F_X_BYTES;
  cudaError_t e = cudaFuncSetAttribute(k5f_mix<LM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k5f_mix<LM><<<(unsigned)p->nmix_fused, K5F_THREADS, smem, s>>>(sp_ld, sp_st, p->d_mix2, p->d_rowoff, p->d_coloff,
                                                                 p->nq, p->d_perm[0], p->d_perm[2], ll, lr, U);
  return cudaGetLastError();
}

cudaError_t launch_pair_mix(const tn_plan* p, const SectorParams& sp1, const double* ll, const double* lr,
                            const double2* U, cudaStream_t s, const SectorParams* sp2_in) {
  const SectorParams& sp2 = sp2_in ? *sp2_in : sp1;   // pass 2 may read one set of buffers and write another
  // The launches touch disjoint elements except pass 2 after pass 1: K5F (its own blocks) runs on an auxiliary
  // stream beside both passes, and each pass's class launches are spread over the caller's stream and two more
  // auxiliary ones (their tails and occupancy overlap, as K5's classes do), joined before pass 2 and at the end.
  // TN_K5_SERIAL=1 keeps everything on the caller's stream.
  static const bool serial = getenv("TN_K5_SERIAL") != nullptr;
  AuxStreams* ap = nullptr;
  if (!serial)
    if (cudaError_t ea = aux_streams(s, &ap); ea != cudaSuccess) return ea;
  cudaStream_t lanes[3] = {s, ap ? ap->st[0] : s, ap ? ap->st[1] : s};
  cudaError_t e = cudaSuccess;
  if (ap) e = cudaEventRecord(ap->fork, s);
  // K5F blocks (both species at once) read P from sp1's buffers and write Θ through sp2's (the same tables for a
  // plain exec; tn_theta_exec_remote: local workspace → the owners' buffers)
  const bool fused_aux = ap && p->nmix_fused > 0;
  if (e == cudaSuccess && fused_aux) e = cudaStreamWaitEvent(ap->st[2], ap->fork, 0);
  if (e == cudaSuccess) e = launch_pair_mix_fused(p, sp1, sp2, ll, lr, U, fused_aux ? ap->st[2] : s);
  if (e == cudaSuccess && fused_aux) e = cudaEventRecord(ap->join[2], ap->st[2]);
  const int Lmax = p->max_mix;
  const int Lc[4] = {std::min(Lmax, 8), std::min(Lmax, 16), std::min(Lmax, 32), Lmax};
  for (int pass = 0; pass < 2 && e == cudaSuccess; ++pass) {
    if (p->nmix2[pass] == 0) continue;
    const MixTile2* tiles = p->d_mix2 + p->nmix_fused + (pass ? p->nmix2[0] : 0);
    const SectorParams& sp = pass ? sp2 : sp1;
    if (ap && pass == 1) e = cudaEventRecord(ap->fork, s);   // pass 2 starts after pass 1 (joined into s)
    bool used[3] = {true, false, false};
    int lane = 0;
    for (int multi = 0; multi < 2 && e == cudaSuccess; ++multi)
      for (int c = 0; c < 4 && e == cudaSuccess; ++c) {
        const int64_t cnt = p->nmix2_grp[pass][multi][c];
        if (cnt == 0) continue;
        const int L = Lc[c], NT = (L + 7) >> 3, smax = mix_us_elems(L), nfix = multi ? p->nfix_max : 1;
        cudaStream_t ls = lanes[lane];
        if (ap && lane > 0 && !used[lane]) {
          e = cudaStreamWaitEvent(ls, ap->fork, 0);
          used[lane] = true;
          if (e != cudaSuccess) break;
        }
        lane = (lane + 1) % 3;
#define TN_P_LAUNCH(M, MULTI)                                                                                 \
  do {                                                                                                        \
    const size_t smem = (size_t)smax * (sizeof(double2) + sizeof(double)) + 2 * 8 * (M) * (size_t)nfix * sizeof(SecRef); \
    if (smem > 48 * 1024) {                                                                                   \
      e = cudaFuncSetAttribute(k5p_mix<M, MULTI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
      if (e != cudaSuccess) return e;                                                                         \
    }                                                                                                         \
    k5p_mix<M, MULTI><<<(unsigned)cnt, K5P_THREADS, smem, ls>>>(sp, tiles, p->d_rowoff, p->d_coloff, p->nq,      \
                                                                p->d_perm[0], p->d_perm[2], ll, lr, U, smax, nfix); \
  } while (0)
#define TN_P_CLASS(M)                    \
  do {                                   \
    if (multi) TN_P_LAUNCH(M, true);     \
    else TN_P_LAUNCH(M, false);          \
  } while (0)
        if (NT <= 1)
          TN_P_CLASS(1);
        else if (NT <= 2)
          TN_P_CLASS(2);
        else if (NT <= 4)
          TN_P_CLASS(4);
        else if (NT <= 6)
          TN_P_CLASS(6);
        else
          TN_P_CLASS(8);
#undef TN_P_CLASS
#undef TN_P_LAUNCH
        tiles += cnt;
        e = cudaGetLastError();
      }
    // join this pass's auxiliary lanes back into s
    for (int k = 1; k < 3 && e == cudaSuccess; ++k)
      if (ap && used[k]) {
        e = cudaEventRecord(ap->join[k - 1], lanes[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ap->join[k - 1], 0);
      }
  }
  if (e == cudaSuccess && fused_aux) e = cudaStreamWaitEvent(s, ap->join[2], 0);
  return e;
}

}  // namespace tn
