// K5T — the U-mix of K5 (Eq. S5's U_n-weighted sum over c_c; see k5_mix.cu for the
// arithmetic) restructured so that HBM only ever sees long contiguous runs, issued by TMA.
//
// Work item = nrows rows × w columns of one (c_l, c_r) block (all L = hi−lo+1 sectors of that block).
// Its data are L·nrows runs of w contiguous complex numbers, one per (row, sector) — each run is one
// 1-D bulk copy (cp.async.bulk) global → shared, and after the mix one bulk copy shared → global.
//
//  * Persistent CTAs, one per SM: warp 8 is the producer, warps 0–7 mix. Items are taken round-robin in
//    row-major order (row band, then c_r, then column chunk), so the CTAs running at any time sweep the
//    same sector rows — the order the access probe (tools/probe_mix_bw.cu) found fastest.
//  * NS-stage ring in shared memory. Producer, per item: wait until the stage's previous item has been
//    mixed (empty barrier, 8 warp arrivals), bulk-store its L·nrows result runs, wait for those stores to
//    finish READING shared memory, then expect_tx + bulk-load the new item's runs, stage its U
//    sub-block (Us[t][u], Re+Im copy) and the per-sector pointer table, and arrive on the full barrier.
//  * Mixer warps: the same DMMA.8x8x4 Gauss 3-product mix as K5 (one 8-column group per warp step,
//    M = 8 columns, K = u, N = t), operands from shared memory, the λl·λr-scaled result written back in
//    place into the stage (a group's columns belong to that group only; every lane's loads complete
//    before the warp's last MMA), then fence.proxy.async so the bulk store sees the writes.
//  * Run stride in shared memory ≡ 32 bytes mod 128, so a quarter-warp A-fragment LDS.128 (2 columns ×
//    4 sectors) covers 32 distinct banks.
//  * The in-place global update is race-free: every element belongs to exactly one item.
// Status: opt-in experiment (TN_K5T=1 at plan time), parity-green but SLOWER than k5_mix: config 3
// 1.65 vs 0.72 ms (1.39 ms even with the U staging removed), config 4 10.5 vs 4.3 ms — one producer
// warp issuing ~1–4 KB bulk copies per (row, sector) run and one CTA per SM do not reach the memory
// parallelism of k5_mix's 16–32 warps of plain loads.
#include "k4_device.cuh"
#include "k5_mix.cuh"

namespace tn {

namespace {
constexpr int K5T_CONS = 8;                       // mixer warps
constexpr int K5T_THREADS = (K5T_CONS + 1) * 32;  // + one producer warp

template <int NT>
struct K5TCfg {
  static constexpr int LMAX = 8 * NT;
  static constexpr int NS = NT >= 4 ? 3 : 4;               // ring stages
  static constexpr int STAGE = 40 * 1024;                  // data bytes per stage
  static constexpr int UP = (LMAX + 3) & ~3;
  static constexpr int UST = ((UP * 16) % 128 == 64) ? UP : UP + 4;  // us_stride(UP)
  static constexpr int US = LMAX * UST;                    // Us entries per stage (TP = LMAX rows)
};

struct K5THdr {                 // per-stage item description (written by the producer)
  const double2* ld[32];        // sector lo+u at (item row 0, item column 0); nullptr: empty segment (P = 0)
  double2* st[32];              // output sector lo+t at the same origin
  int64_t ldd[32];              // row stride (elements) of sector lo+u (items have L ≤ 32)
  int32_t L, nrows, w, stride;  // stride: elements per shared-memory run
  int32_t ust, pl, pc;          // Us row stride; sorted position of row 0 / column 0
  int32_t pad;
};

__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace

template <int NT>
__global__ void __launch_bounds__(K5T_THREADS, 1)
    k5t_mix(const SectorParams sp, const MixItem* __restrict__ items, int nitems, const int32_t* __restrict__ perm_l,
            const int32_t* __restrict__ perm_r, const double* __restrict__ ll, const double* __restrict__ lr,
            const double2* __restrict__ U) {
  using C = K5TCfg<NT>;
  constexpr int NS = C::NS, KSM = 2 * NT;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* data = smem_raw;                                                     // NS × STAGE
  double2* Usb = reinterpret_cast<double2*>(data + (size_t)NS * C::STAGE);     // NS × US
  double* UsSb = reinterpret_cast<double*>(Usb + (size_t)NS * C::US);          // NS × US
  K5THdr* hdr = reinterpret_cast<K5THdr*>(UsSb + (size_t)NS * C::US);          // NS
  uint64_t* full = reinterpret_cast<uint64_t*>(hdr + NS);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, K5T_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int d = sp.d;
  if (warp == K5T_CONS) {
    // ------------------------------------------------ producer ------------------------------------------------
    int k = 0;
    auto store_stage = [&](int s) {  // bulk-store the mixed runs of the item held in stage s (lane 0)
      const K5THdr& H = hdr[s];
      const uint8_t* base = data + (size_t)s * C::STAGE;
      for (int x = lane; x < H.nrows * H.L; x += 32) {
        const int r = x / H.L, t = x - r * H.L;
        bulk_s2g(H.st[t] + (int64_t)r * H.ldd[t], base + (size_t)x * H.stride * 16, (uint32_t)H.w * 16);
      }
      bulk_commit();
      bulk_wait_read0();
      __syncwarp();
    };
    for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++k) {
      const int s = k % NS;
      if (k >= NS) {
        mbar_wait(empty + s, ((k / NS) - 1) & 1);
        store_stage(s);
      }
      const MixItem I = items[it];
      const int c_l = I.cl, c_r = I.cr, n = c_l - c_r;
      const int lo = max(c_r, c_l - d + 1), hi = min(c_l, c_r + d - 1), L = hi - lo + 1;
      const int stride = I.stride;
      K5THdr& H = hdr[s];
      uint32_t bytes = 0;
      for (int u = 0; u < L; ++u) {  // uniform per warp: every lane computes the table, lane u % 32 writes it
        const int cc = lo + u;
        const int64_t off = ((int64_t)I.pl - sp.lrow0[cc]) * sp.ld[cc] + ((int64_t)I.pc - sp.col0[cc]);
        const bool ne = (sp.cc_mask[cc >> 5] >> (cc & 31)) & 1u;
        if (ne) bytes += (uint32_t)(I.nrows * I.w * 16);
        if ((u & 31) == lane) {
          H.ld[u] = ne ? (sp.src[cc] ? sp.src[cc] + off : sp.out[cc] + off) : nullptr;
          H.st[u] = sp.out[cc] + off;
          H.ldd[u] = sp.ld[cc];
        }
      }
      if (lane == 0) {
        H.L = L;
        H.nrows = I.nrows;
        H.w = I.w;
        H.stride = stride;
        H.ust = C::UST;
        H.pl = I.pl;
        H.pc = I.pc;
        if (bytes) mbar_expect_tx_only(full + s, bytes);
      }
      __syncwarp();
      uint8_t* base = data + (size_t)s * C::STAGE;
      for (int x = lane; x < I.nrows * L; x += 32) {
        const int r = x / L, u = x - r * L;
        const double2* src = H.ld[u];
        if (src) bulk_g2s(base + (size_t)x * stride * 16, src + (int64_t)r * H.ldd[u], (uint32_t)I.w * 16, full + s);
      }
      // Us[t][u] = U_n[c_l − (lo+t)][c_l − (lo+u)], zero-padded to LMAX × UP
      const int nlo = max(0, n - d + 1), sn = min(n, d - 1) - nlo + 1;
      const double2* Ub = U + sp.ustart[n];
      double2* Us = Usb + (size_t)s * C::US;
      double* UsS = UsSb + (size_t)s * C::US;
      const int TP = (L + 7) & ~7;
      for (int x = lane; x < TP * C::UP; x += 32) {
        const int t = x / C::UP, u = x - t * C::UP;
        double2 v = make_double2(0.0, 0.0);
        if (t < L && u < L) v = __ldg(Ub + (c_l - lo - t - nlo) * sn + (c_l - lo - u - nlo));
        Us[t * C::UST + u] = v;
        UsS[t * C::UST + u] = v.x + v.y;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(full + s);
    }
    // drain: store the last min(NS, k) items
    for (int j = max(0, k - NS); j < k; ++j) {
      const int s = j % NS;
      mbar_wait(empty + s, (j / NS) & 1);
      store_stage(s);
    }
    bulk_wait0();  // every lane's bulk stores complete before the CTA exits
    return;
  }
  // ---------------------------------------------------- mixers ----------------------------------------------------
  const int g = lane >> 2, q = lane & 3;
  int k = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++k) {
    const int s = k % NS;
    mbar_wait(full + s, (k / NS) & 1);
    const K5THdr& H = hdr[s];
    const int L = H.L, nrows = H.nrows, w = H.w, stride = H.stride;
    const int KS = (L + 3) >> 2, TPn = (L + 7) >> 3;
    double2* base = reinterpret_cast<double2*>(data + (size_t)s * C::STAGE);
    const double2* Us = Usb + (size_t)s * C::US;
    const double* UsS = UsSb + (size_t)s * C::US;
    bool ldok[KSM];
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) {
      const int u = ks * 4 + q;
      ldok[ks] = u < L && H.ld[u] != nullptr;
    }
    const int ngr = (w + 7) >> 3, G = nrows * ngr;
    for (int grp = warp; grp < G; grp += K5T_CONS) {
      const int r = grp / ngr, col = (grp - r * ngr) * 8 + g;
      const bool valid = col < w;
      double2* row = base + (size_t)r * L * stride + col;
      double2 a[KSM];
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) {
        a[ks] = make_double2(0.0, 0.0);
        if (ks < KS && valid && ldok[ks]) a[ks] = row[(size_t)(ks * 4 + q) * stride];
      }
      double acc[NT][6];
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int x = 0; x < 6; ++x) acc[j][x] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) {
        if (ks < KS) {
          const double as = a[ks].x + a[ks].y;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            if (j < TPn) {
              const int idx = (j * 8 + g) * C::UST + ks * 4 + q;
              const double2 b = Us[idx];
              const double bs = UsS[idx];
              dmma5(acc[j][0], acc[j][1], a[ks].x, b.x);
              dmma5(acc[j][2], acc[j][3], a[ks].y, b.y);
              dmma5(acc[j][4], acc[j][5], as, bs);
            }
          }
        }
      }
      if (valid) {
        const double scale = ll[perm_l[H.pl + r]] * lr[perm_r[H.pc + col]];
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = j * 8 + 2 * q + h;
            if (j < TPn && t < L) {
              const double re = acc[j][h] - acc[j][2 + h];
              const double im = acc[j][4 + h] - acc[j][h] - acc[j][2 + h];
              row[(size_t)t * stride] = make_double2(re * scale, im * scale);
            }
          }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
}

template <int NT>
size_t k5t_smem() {
  using C = K5TCfg<NT>;
  return (size_t)C::NS * C::STAGE + (size_t)C::NS * C::US * (sizeof(double2) + sizeof(double)) +
         (size_t)C::NS * sizeof(K5THdr) + 2 * C::NS * sizeof(uint64_t);
}

// shared-memory run stride (elements) for w columns: ≡ 32 bytes mod 128
inline int k5t_stride(int w) { return ((w * 16 + 127) / 128 * 128 + 32) / 16; }

// Items for the blocks with L ≤ 32, in row-major order (8-row bands, then c_r, then row sub-band, then
// column chunk), one list per register class (L ≤ 8, ≤ 16, ≤ 32); w and nrows fill one ring stage.
void build_mix_items(tn_plan* p, std::vector<MixItem>& out) {
  out.clear();
  std::vector<MixItem> cls[3];
  const auto& ol = p->off[0];
  const auto& orr = p->off[2];
  constexpr int BANDR = 8;
  const int stage = K5TCfg<1>::STAGE;
  for (int cl = 0; cl <= p->N; ++cl) {
    const int64_t a0 = std::max<int64_t>(ol[cl], p->r0), a1 = std::min<int64_t>(ol[cl + 1], p->r1);
    for (int64_t band = a0; band < a1; band += BANDR) {
      const int64_t brows = std::min<int64_t>(BANDR, a1 - band);
      for (int cr = std::max(0, cl - 2 * p->d + 2); cr <= cl; ++cr) {
        const int nr = orr[cr + 1] - orr[cr];
        if (nr == 0) continue;
        const int L = std::min(cl, cr + p->d - 1) - std::max(cr, cl - p->d + 1) + 1;
        if (L > 32) continue;
        const int c = L <= 8 ? 0 : L <= 16 ? 1 : 2;
        int w = std::min(nr, 256);
        while (w > 8 && (int64_t)L * k5t_stride(w) * 16 > stage) w -= 8;
        const int nrows = (int)std::max<int64_t>(1, std::min<int64_t>(brows, stage / ((int64_t)L * k5t_stride(w) * 16)));
        for (int64_t r0 = band; r0 < band + brows; r0 += nrows)
          for (int j0 = 0; j0 < nr; j0 += w) {
            MixItem I;
            I.cl = cl;
            I.cr = cr;
            I.pl = (int32_t)r0;
            I.nrows = (int32_t)std::min<int64_t>(nrows, band + brows - r0);
            I.pc = orr[cr] + j0;
            I.w = std::min(w, nr - j0);
            I.stride = k5t_stride(I.w);
            I.pad = 0;
            cls[c].push_back(I);
          }
      }
    }
  }
  for (int c = 0; c < 3; ++c) {
    p->nitem_cls[c] = (int64_t)cls[c].size();
    out.insert(out.end(), cls[c].begin(), cls[c].end());
  }
}

// K5T for the L ≤ 32 blocks (three persistent launches), k5_mix for the rest. Returns false (nothing
// launched) when K5T does not apply: remote exec (P read from a workspace, Θ possibly in peer memory).
cudaError_t launch_mix_tma(const tn_plan* p, const SectorParams& sp, const double* ll, const double* lr,
                           const double2* U, cudaStream_t s) {
  const MixItem* it = p->d_items;
  cudaError_t e = cudaSuccess;
#define TN_K5T(NTv, n)                                                                                    \
  do {                                                                                                    \
    if ((n) > 0 && e == cudaSuccess) {                                                                    \
      const size_t smem = k5t_smem<NTv>();                                                                \
      e = cudaFuncSetAttribute(k5t_mix<NTv>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
      if (e == cudaSuccess) {                                                                             \
        const int grid = (int)std::min<int64_t>((n), p->sm_count);                                        \
        k5t_mix<NTv><<<grid, K5T_THREADS, smem, s>>>(sp, it, (int)(n), p->d_perm[0], p->d_perm[2], ll, lr, U); \
        e = cudaGetLastError();                                                                           \
      }                                                                                                   \
      it += (n);                                                                                          \
    }                                                                                                     \
  } while (0)
  TN_K5T(1, p->nitem_cls[0]);
  TN_K5T(2, p->nitem_cls[1]);
  TN_K5T(4, p->nitem_cls[2]);
#undef TN_K5T
  return e;
}

}  // namespace tn
