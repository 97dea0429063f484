// SVD step after Θ: per-sector SVD, global top-χ, new canonical factors.
//
// PAPER.md:67 "Singular value decompositions are then performed on Θ(c^{[k]}), and the largest χ singular
// values out of the singular values for all Θ(c^{[k]}) and their corresponding bonds are retained";
// PAPER.md:192 (SVD "takes up the majority" of GPU time); contract SPEC.md:70-78, tie-break SPEC.md:97.
//
// B200 design (DESIGN.md §4 "SVD step"):
//  * Per-sector spectrum by default from the Gram eigensolver + Rayleigh–Ritz path (only the
//    values that can enter the global top χ are computed exactly); a full cuSOLVER SVD per sector
//    (polar-decomposition Xgesvdp with TN_SVD_ALGO=gesvdp, one-sided Jacobi gesvdj with TN_SVD_ALGO=gesvdj)
//    is selectable — the SVD itself being a library routine, as the paper treats it ("a well-researched
//    and optimized routine"). Sectors run concurrently on 8 lanes (handle + stream + host
//    thread each), largest first onto the least-loaded lane. Θ(c) is row-major, i.e. the column-major
//    C×R matrix X = Θᵀ = U_x S V_xᴴ, so Θ = conj(V_x) S U_xᵀ.
//  * Global ranking on the device: one stable radix sort (cub) of all singular values, descending, whose
//    input order is (charge asc, index asc) — exactly SPEC.md:97's tie-break; the kept set is a prefix.
//  * K_sel (one CTA): kept count per charge, discarded weight Σ dropped s², new-bond offsets (charge
//    ascending, then value descending = a prefix of every sector's spectrum), q_new and λ_new.
//  * K_fac: Γ^{[k]}_new[α, a] = U_c[α, s]/λl[α] and Γ^{[k+1]}_new[a, β] = V_c†[s, β]/λr[β] (x/0 := 0),
//    written straight into the caller's bond order through perm_l / perm_r.
#include <cub/device/device_radix_sort.cuh>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "tn_internal.cuh"

namespace tn {

namespace {
constexpr int SVD_LANES = 8;  // concurrent sector SVDs (one cuSOLVER handle + stream + host thread each)
struct SvdCtx {  // cuSOLVER handles / streams + a grow-only device scratch, per process and bound to the
                 // device current at first use (one process per GPU, as everywhere in this library)
  cusolverDnHandle_t h[SVD_LANES] = {};
  cublasHandle_t hb[SVD_LANES] = {};
  cudaStream_t st[SVD_LANES] = {};
  cudaEvent_t ev[SVD_LANES + 1] = {};
  gesvdjInfo_t params = nullptr;
  gesvdjInfo_t pj[SVD_LANES] = {};  // per-lane Jacobi settings (the info object also carries results)
  cusolverDnParams_t xparams = nullptr;
  void* buf = nullptr;   // common scratch (library-SVD outputs, ranking buffers)
  size_t cap = 0;
  void* gbuf[3] = {};    // Gram path: phase A (Gram matrices → eigenvectors), phase C (Ritz SVDs), tests
  size_t gcap[3] = {};
  std::mutex mu;
};
SvdCtx& ctx() {
  static SvdCtx c;
  return c;
}
// 2 (default): Gram eigensolver + Rayleigh–Ritz (svd_gram below; 0.26–0.30 s at config 3), 1: polar-decomposition
// SVD per sector (TN_SVD_ALGO=gesvdp, 0.77 s), 0: one-sided Jacobi (TN_SVD_ALGO=gesvdj, 1.98 s); all three
// meet the parity bar (tests/test_gpu_svd.py runs each)
int svd_algo() {
  const char* e = getenv("TN_SVD_ALGO");
  if (e && std::string(e) == "gesvdj") return 0;
  if (e && std::string(e) == "gesvdp") return 1;
  return 2;
}
// largest h_err_sigma accepted from Xgesvdp (Ritz step and TN_SVD_ALGO=gesvdp) before Jacobi redoes it:
// healthy config-2/3 sectors report 0 … 3.9e-13, the failure seen on small rank-deficient sectors 5.1e-8
constexpr double kRitzHerrMax = 1e-11;
tn_status grow(void*& buf, size_t& cap, size_t need, char** out) {  // grow-only device scratch
  if (need > cap) {
    // 25% headroom: the sector shapes of consecutive gates differ, and every regrowth is a synchronising
    // cudaFree + cudaMalloc on the gate's critical path
    const size_t want = need + need / 4;
    if (buf) cudaFree(buf);
    buf = nullptr;
    cap = 0;
    if (cudaMalloc(&buf, want) != cudaSuccess) {
      cudaGetLastError();
      if (cudaMalloc(&buf, need) != cudaSuccess) return fail(TN_ERR_OOM, "tn_svd_truncate: scratch allocation");
      cap = need;
    } else {
      cap = want;
    }
  }
  *out = static_cast<char*>(buf);
  return TN_OK;
}
}  // namespace

struct SvdSector {          // device views of one sector's SVD
  const double2* ux;        // C × k column-major (ld C)
  const double2* vx;        // R × k column-major (ld R)
  const double* s;          // k values, descending
  int64_t row0, col0;       // sorted positions of Θ(c)'s first row / column (single-charge plans)
  const int32_t* rpos;      // pair plans: sorted position of every row / column of Θ(c) (else nullptr:
  const int32_t* cpos;      //   rows row0 + r, columns col0 + j)
  int32_t R, C, k;
};

constexpr int SVD_MAXSEC = MAXC;
struct SvdParams {
  SvdSector sec[SVD_MAXSEC];
  int nsec;
};

struct ThetaPtrs {          // the sectors' device pointers and element counts (kernel parameter)
  const double2* p[SVD_MAXSEC];
  int64_t n[SVD_MAXSEC];
};

// Frobenius² of every sector (blockIdx.y): the largest singular value of Θ(c) is ≤ ‖Θ(c)‖_F, which lets
// the SVD skip sectors that cannot reach the global top χ (their whole weight is discarded)
__global__ void k_sector_norm2(const ThetaPtrs tp, double* __restrict__ out) {
  const int c = blockIdx.y;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tp.n[c]; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = tp.p[c][i];
    acc += v.x * v.x + v.y * v.y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(out + c, acc);
}

__global__ void k_svd_pack(const SvdParams sp, double* __restrict__ keys, int32_t* __restrict__ vals,
                           const int64_t* __restrict__ base) {
  const int c = blockIdx.y;
  const SvdSector S = sp.sec[c];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S.k; i += gridDim.x * blockDim.x) {
    keys[base[c] + i] = S.s[i];
    vals[base[c] + i] = (c << 20) | i;  // k < 2^20 (χ ≤ INT32 and sectors ≤ 2^20 columns)
  }
}

__global__ void __launch_bounds__(1024) k_svd_select(const SvdParams sp, const double* __restrict__ skeys,
                                                      const int32_t* __restrict__ svals, int64_t total,
                                                      int64_t chi_max, double cutoff, int32_t* __restrict__ q_new,
                                                      double* __restrict__ lam_new, int32_t* __restrict__ off_new,
                                                      int64_t* __restrict__ chi_out, double* __restrict__ disc_out,
                                                      double disc_extra) {
  __shared__ int32_t kept[SVD_MAXSEC + 1];
  __shared__ double red[32];
  __shared__ int64_t nkeep_s;
  const int tid = threadIdx.x;
  for (int c = tid; c <= SVD_MAXSEC; c += blockDim.x) kept[c] = 0;
  if (tid == 0) {
    // kept = the first min(chi_max, #(s > cutoff)) sorted entries (values > cutoff form a prefix)
    int64_t lo = 0, hi = total;  // first index with s ≤ cutoff
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (skeys[mid] > cutoff) lo = mid + 1;
      else hi = mid;
    }
    nkeep_s = lo < chi_max ? lo : chi_max;
  }
  __syncthreads();
  const int64_t nkeep = nkeep_s;
  double acc = 0.0;
  for (int64_t i = tid; i < total; i += blockDim.x) {
    if (i < nkeep) atomicAdd(&kept[svals[i] >> 20], 1);
    else acc += skeys[i] * skeys[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *disc_out = t + disc_extra;  // + the whole weight of sectors skipped by the norm bound
    *chi_out = nkeep;
    int32_t o = 0;
    for (int c = 0; c < sp.nsec; ++c) {
      off_new[c] = o;
      o += kept[c];
    }
    off_new[sp.nsec] = o;
  }
  __syncthreads();
  for (int c = 0; c < sp.nsec; ++c) {  // new bond a = off_new[c] + s, s < kept[c]
    const int32_t o = off_new[c];
    for (int s = tid; s < kept[c]; s += blockDim.x) {
      q_new[o + s] = c;
      lam_new[o + s] = sp.sec[c].s[s];
    }
  }
}

// blockIdx.y = sector; Γk_new rows (α of Θ(c)) × kept columns, then Γk1_new kept rows × columns (β)
__global__ void k_svd_factors(const SvdParams sp, const int32_t* __restrict__ off_new, const int32_t* __restrict__ perm_l,
                              const int32_t* __restrict__ perm_r, const double* __restrict__ lam_l,
                              const double* __restrict__ lam_r, int64_t ld_k, int64_t chi_r,
                              double2* __restrict__ gk_new, double2* __restrict__ gk1_new) {
  const int c = blockIdx.y;
  const SvdSector S = sp.sec[c];
  const int32_t a0 = off_new[c], kc = off_new[c + 1] - a0;
  if (kc == 0) return;
  const int64_t na = (int64_t)S.R * kc, nb = (int64_t)kc * S.C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < na) {  // U_Θ[r, s] = conj(V_x[r, s]); consecutive threads → consecutive new-bond columns
      const int r = (int)(i / kc), s = (int)(i - (int64_t)r * kc);
      const int32_t al = perm_l[S.rpos ? (int64_t)S.rpos[r] : S.row0 + r];
      const double l = lam_l[al];
      const double2 v = S.vx[r + (int64_t)s * S.R];
      const double inv = l != 0.0 ? 1.0 / l : 0.0;
      gk_new[(int64_t)al * ld_k + a0 + s] = make_double2(v.x * inv, -v.y * inv);
    } else {       // V_Θ†[s, col] = U_x[col, s]
      const int64_t j = i - na;
      const int s = (int)(j / S.C), col = (int)(j - (int64_t)s * S.C);
      const int32_t be = perm_r[S.cpos ? (int64_t)S.cpos[col] : S.col0 + col];
      const double l = lam_r[be];
      const double2 u = S.ux[col + (int64_t)s * S.C];
      const double inv = l != 0.0 ? 1.0 / l : 0.0;
      gk1_new[(int64_t)(a0 + s) * chi_r + be] = make_double2(u.x * inv, u.y * inv);
    }
  }
}

struct BformPtrs {          // per sector: T = (Θ(c)·V_c)ᵀ, kept-count × R column-major (ld = kept count)
  const double2* t[SVD_MAXSEC];
};

// right-canonical factors (R22): B^{[k]}_new[α, a0+s] = T[s, r] / λl[α] (x/0 := 0), B^{[k+1]}_new[a0+s, β]
// = V_Θ†[s, col] = U_x[col, s]
__global__ void k_svd_bform(const SvdParams sp, const BformPtrs bp, const int32_t* __restrict__ off_new,
                            const int32_t* __restrict__ perm_l, const int32_t* __restrict__ perm_r,
                            const double* __restrict__ lam_l, int64_t ld_k, int64_t chi_r, double2* __restrict__ bk_new,
                            double2* __restrict__ bk1_new) {
  const int c = blockIdx.y;
  const SvdSector S = sp.sec[c];
  const int32_t a0 = off_new[c], kc = off_new[c + 1] - a0;
  if (kc == 0) return;
  const int64_t na = (int64_t)S.R * kc, nb = (int64_t)kc * S.C;
  const double2* T = bp.t[c];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < na) {
      const int r = (int)(i / kc), s = (int)(i - (int64_t)r * kc);
      const int32_t al = perm_l[S.rpos ? (int64_t)S.rpos[r] : S.row0 + r];
      const double l = lam_l[al];
      const double2 v = T[s + (int64_t)r * kc];
      bk_new[(int64_t)al * ld_k + a0 + s] = l != 0.0 ? make_double2(v.x / l, v.y / l) : make_double2(0.0, 0.0);
    } else {
      const int64_t j = i - na;
      const int s = (int)(j / S.C), col = (int)(j - (int64_t)s * S.C);
      const int32_t be = perm_r[S.cpos ? (int64_t)S.cpos[col] : S.col0 + col];
      bk1_new[(int64_t)(a0 + s) * chi_r + be] = S.ux[col + (int64_t)s * S.C];
    }
  }
}

// ---- Ritz refinement (phase C of the Gram path, DESIGN.md §4 "SVD step") ----
// Y = Z·E_k' has nearly orthogonal columns (E_k' are eigenvectors of ZᴴZ): with M = YᴴY, the scaled coupling
// ρ_ij = |M_ij| / √(M_ii M_jj) is ~ ε·w_max / w at worst (the eigenvectors' backward error). Instead of a full SVD
// of Y, each pass rotates every column pair (i, j) by the exact 2×2 Jacobi rotation of [[M_ii, M_ij], [M_ji,
// M_jj]], all pairs at once (V = I + the rotations' off-diagonal entries): first order in ρ, so a pass squares ρ
// and the second pass finds it at rounding level. The scaled convergence test is the one-sided Jacobi criterion
// (Demmel–Veselić), so the column norms of the rotated Y are the Ritz values to relative rounding accuracy.

// V[i + j·k] for column-major M (k × k); atomically records max ρ over the off-diagonal pairs (bit pattern of a
// non-negative double orders like an unsigned integer)
__global__ void k_ritz_rot(const double2* __restrict__ M, int k, double2* __restrict__ V,
                           unsigned long long* __restrict__ rho_max) {
  double rho = 0.0;
  const int64_t kk = (int64_t)k * k;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < kk; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x % k), j = (int)(x / k);
    if (i == j) {
      V[x] = make_double2(1.0, 0.0);
      if (!(M[x].x > 0.0)) rho = INFINITY;   // a zero column has no direction to refine: library SVD
      continue;
    }
    const double a = M[i + (int64_t)i * k].x, d = M[j + (int64_t)j * k].x;
    const double2 b = M[x];                      // M_ij = y_iᴴ y_j
    const double ab = hypot(b.x, b.y);
    double2 v = make_double2(0.0, 0.0);
    if (ab > 0.0) {
      const double den = sqrt(fmax(a, 0.0)) * sqrt(fmax(d, 0.0));
      rho = fmax(rho, den > 0.0 ? ab / den : INFINITY);
      // v_j's i-th component: s·b/|b| with t = tan θ the smaller root of the 2×2 problem (|θ| ≤ π/4);
      // to first order b / (M_jj − M_ii)
      const double zeta = (d - a) / (2.0 * ab);
      const double az = fabs(zeta);
      const double r = az > 1.0 ? az * sqrt(1.0 + 1.0 / (az * az)) : sqrt(1.0 + az * az);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (az + r);
      const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
      v = make_double2(s * b.x / ab, s * b.y / ab);
    }
    V[x] = v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) rho = fmax(rho, __shfl_xor_sync(0xffffffffu, rho, o));
  if ((threadIdx.x & 31) == 0 && rho > 0.0) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(rho);
    atomicMax(rho_max, bits);
  }
}

__global__ void k_eye(double2* __restrict__ W, int k, double alpha, double beta) {  // W ← α·I + β·W
  const int64_t kk = (int64_t)k * k;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < kk; x += (int64_t)gridDim.x * blockDim.x) {
    const double2 w = beta != 0.0 ? W[x] : make_double2(0.0, 0.0);
    const double e = (x % k) == (x / k) ? alpha : 0.0;
    W[x] = make_double2(e + beta * w.x, beta * w.y);
  }
}

// s²_j = ‖Y[:, j]‖² (one block per column; Y column-major, ld m)
__global__ void k_colnorm2(const double2* __restrict__ Y, int64_t m, double* __restrict__ s2) {
  const int j = blockIdx.x;
  const double2* y = Y + (int64_t)j * m;
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) acc += y[r].x * y[r].x + y[r].y * y[r].y;
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    s2[j] = t;
  }
}

// descending order of s² (ties: lower column first): src[rank] = column
__global__ void k_ritz_rank(const double* __restrict__ s2, int k, int32_t* __restrict__ src) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double v = s2[i];
  int r = 0;
  for (int j = 0; j < k; ++j) {
    const double u = s2[j];
    r += (u > v) || (u == v && j < i);
  }
  src[r] = i;
}

// P[:, r] = Y[:, src[r]] / s, Wout[:, r] = W[:, src[r]], S[r] = s = √s²[src[r]]
__global__ void k_ritz_permute(const double2* __restrict__ Y, const double2* __restrict__ W,
                               const double* __restrict__ s2, const int32_t* __restrict__ src, int64_t m, int k,
                               double2* __restrict__ P, double2* __restrict__ Wout, double* __restrict__ S) {
  const int64_t ny = m * k, nw = (int64_t)k * k;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < ny + nw + k;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x < ny) {
      const int r = (int)(x / m);
      const int64_t row = x - (int64_t)r * m;
      const int j = src[r];
      const double s = sqrt(s2[j]);
      const double inv = s > 0.0 ? 1.0 / s : 0.0;
      const double2 y = Y[row + (int64_t)j * m];
      P[x] = make_double2(y.x * inv, y.y * inv);
    } else if (x < ny + nw) {
      const int64_t z = x - ny;
      const int r = (int)(z / k);
      const int64_t row = z - (int64_t)r * k;
      Wout[z] = W[row + (int64_t)src[r] * k];
    } else {
      const int r = (int)(x - ny - nw);
      S[r] = sqrt(s2[src[r]]);
    }
  }
}

// Run job(lane, c, host_workspace) for every sector of `wave` on the SVD lanes (largest cost first onto the
// least-loaded lane; one host thread per lane, each lane's stream joined back into `s`).
template <class Cost, class Job>
tn_status run_lanes(SvdCtx& X, cudaStream_t s, std::vector<int> wave, Cost cost, Job job) {
  if (wave.empty()) return TN_OK;
  std::sort(wave.begin(), wave.end(), [&](int a, int b) { return cost(a) > cost(b); });
  std::vector<std::vector<int>> lane(SVD_LANES);
  double load[SVD_LANES] = {};
  for (int c : wave) {
    const int l = (int)(std::min_element(load, load + SVD_LANES) - load);
    lane[l].push_back(c);
    load[l] += cost(c);
  }
  tn_status r0 = cuda_check(cudaEventRecord(X.ev[SVD_LANES], s), "Θ ready");
  if (r0 != TN_OK) return r0;
  std::vector<std::string> errs(SVD_LANES);
  int dev = 0;
  cudaGetDevice(&dev);   // lane threads must run on the caller's device (one process per GPU, any local rank)
  auto work = [&](int l) {
    if (lane[l].empty()) return;
    if (cudaSetDevice(dev) != cudaSuccess) {
      errs[l] = "set device";
      return;
    }
    if (cudaStreamWaitEvent(X.st[l], X.ev[SVD_LANES], 0) != cudaSuccess) {
      errs[l] = "stream wait";
      return;
    }
    std::vector<char> hbuf;
    for (int c : lane[l]) {
      errs[l] = job(l, c, hbuf);
      if (!errs[l].empty()) return;
    }
    if (cudaEventRecord(X.ev[l], X.st[l]) != cudaSuccess) errs[l] = "event record";
  };
  {
    std::vector<std::thread> th;
    for (int l = 1; l < SVD_LANES; ++l) th.emplace_back(work, l);
    work(0);
    for (auto& t : th) t.join();
  }
  for (int l = 0; l < SVD_LANES; ++l) {
    if (!errs[l].empty()) return fail(TN_ERR_CUDA, "tn_svd_truncate: " + errs[l]);
    if (!lane[l].empty() && (r0 = cuda_check(cudaStreamWaitEvent(s, X.ev[l], 0), "join SVD lanes")) != TN_OK) return r0;
  }
  return TN_OK;
}

// ---- Gram eigensolver + Rayleigh–Ritz SVD step (default) ----
// The column-major view of Θ(c) is Z = Θᵀ (C × R, ld C). With n_g = min(R, C):
//  A. G = ZᴴZ (R ≤ C, "tall") or ZZᴴ (R > C), n_g × n_g, by ZGEMM on the DMMA pipe; Hermitian eigensolver
//     (Xsyevd): eigenvalues w ≈ s² with absolute error ≲ n_g·ε·‖G‖, eigenvectors E (ascending).
//  B. (host) approximate global χ-th value T² from every sector's w; a sector keeps its k' top eigenvectors
//     with w ≥ T² − 2Δ (Δ = the largest error bound 16·n_g·ε·w_max over sectors) and w ≥ cutoff² − Δ_c, so
//     every value that can make the exact top χ (or pass the cutoff) is inside E_k'. The norm bound of the
//     library path skips whole sectors the same way (‖Θ(c)‖²_F < T² − Δ).
//  C. Rayleigh–Ritz: Y = Z·E_k' (tall) or Zᴴ·E_k' (max(R,C) × k', ZGEMM), exact SVD Y = P S Wᴴ — by the Ritz
//     refinement (simultaneous 2×2 Jacobi rotations of Y's nearly orthogonal columns until the scaled coupling is at
//     rounding level, k_ritz_rot; falls back to a library SVD of Y when it does not converge, e.g. kept values
//     below the Gram matrix's resolution) — then Z ≈ P S (E_k' W)ᴴ (tall) or (E_k' W) S Pᴴ. Ritz values are accurate to second order in the
//     subspace error, i.e. to ~ε relative, and both factors are orthonormal to ~ε. The weight outside the
//     computed values, ‖Θ(c)‖²_F − Σ S², joins the discarded weight. Θ(c) is read, not destroyed.
tn_status svd_gram(SvdCtx& X, cudaStream_t s, double* const* theta, SvdParams& sp, const std::vector<double>& n2,
                   const std::vector<int>& wave1, const std::vector<int>& rest, int64_t chi_max, double cutoff,
                   double& disc_skipped) {
  const int ns = sp.nsec;
  struct Geo {
    int R, C, ng, mt;
    bool tall;
  };
  std::vector<Geo> g(ns);
  for (int c = 0; c < ns; ++c) {
    const int R = sp.sec[c].R, C = sp.sec[c].C;
    const bool tall = C >= R;
    g[c] = Geo{R, C, tall ? R : C, tall ? C : R, tall};
  }
  auto cost = [&](int c) { return (double)g[c].ng * g[c].ng * ((double)g[c].mt + 3.0 * g[c].ng); };
  // phase-A scratch for every candidate sector
  std::vector<size_t> oG(ns, 0), oW(ns, 0), oWs(ns, 0), wsA(ns, 0), hsA(ns, 0);
  // eigenpairs computed per sector (ascending, the top of the spectrum): n_g with Xsyevd, or only those ≥ vlo[c]
  // with the ranged Xsyevdx (wave 2: the values that can still reach the top χ, DESIGN.md §4 "SVD step")
  std::vector<int64_t> nw(ns, 0);
  std::vector<double> vlo(ns, -1.0);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  std::vector<int> cand(wave1);
  cand.insert(cand.end(), rest.begin(), rest.end());
  for (int c : cand) {
    const int64_t n = g[c].ng;
    if (cusolverDnXsyevd_bufferSize(X.h[0], X.xparams, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F,
                                    nullptr, n, CUDA_R_64F, nullptr, CUDA_C_64F, &wsA[c], &hsA[c]) !=
        CUSOLVER_STATUS_SUCCESS)
      return fail(TN_ERR_CUDA, "cusolverDnXsyevd_bufferSize failed");
    {
      double vl = 0.0, vu = 1.0;
      int64_t m = 0;
      size_t wx = 0, hx = 0;
      if (cusolverDnXsyevdx_bufferSize(X.h[0], X.xparams, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_V,
                                       CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, nullptr, n, &vl, &vu, 0, 0, &m, CUDA_R_64F,
                                       nullptr, CUDA_C_64F, &wx, &hx) != CUSOLVER_STATUS_SUCCESS)
        return fail(TN_ERR_CUDA, "cusolverDnXsyevdx_bufferSize failed");
      wsA[c] = std::max(wsA[c], wx);
      hsA[c] = std::max(hsA[c], hx);
    }
    oG[c] = take((size_t)n * n * 16);
    oW[c] = take((size_t)n * 8);
    oWs[c] = take(wsA[c]);
  }
  const size_t oInfo = take((size_t)2 * ns * 4);
  char* A = nullptr;
  tn_status st = grow(X.gbuf[0], X.gcap[0], off, &A);
  if (st != TN_OK) return st;
  int* infoA = reinterpret_cast<int*>(A + oInfo);
  int* infoC = infoA + ns;
  if ((st = cuda_check(cudaMemsetAsync(infoA, 0, 2 * ns * sizeof(int), s), "memset info")) != TN_OK) return st;
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  auto gram = [&](int l, int c) -> std::string {
    const Geo& q = g[c];
    const auto* Z = reinterpret_cast<const cuDoubleComplex*>(theta[c]);
    auto* G = reinterpret_cast<cuDoubleComplex*>(A + oG[c]);
    const cublasStatus_t b =
        q.tall ? cublasZgemm(X.hb[l], CUBLAS_OP_C, CUBLAS_OP_N, q.R, q.R, q.C, &one, Z, q.C, Z, q.C, &zero, G, q.R)
               : cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_C, q.C, q.C, q.R, &one, Z, q.C, Z, q.C, &zero, G, q.C);
    return b == CUBLAS_STATUS_SUCCESS ? std::string() : "cuBLAS Gram matrix failed in sector " + std::to_string(c);
  };
  auto eig = [&](int l, int c, std::vector<char>& hbuf) -> std::string {
    const Geo& q = g[c];
    hbuf.resize(std::max<size_t>(hsA[c], 1));
    cusolverStatus_t r;
    if (vlo[c] > 0.0) {
      // only the eigenvalues ≥ vlo (they land in the first m columns / entries, ascending)
      double vl = vlo[c], vu = std::numeric_limits<double>::max();
      int64_t m = 0;
      r = cusolverDnXsyevdx(X.h[l], X.xparams, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_V, CUBLAS_FILL_MODE_LOWER,
                            q.ng, CUDA_C_64F, A + oG[c], q.ng, &vl, &vu, 0, 0, &m, CUDA_R_64F, A + oW[c], CUDA_C_64F,
                            A + oWs[c], wsA[c], hbuf.data(), hsA[c], infoA + c);
      nw[c] = m;
    } else {
      r = cusolverDnXsyevd(X.h[l], X.xparams, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, q.ng, CUDA_C_64F,
                           A + oG[c], q.ng, CUDA_R_64F, A + oW[c], CUDA_C_64F, A + oWs[c], wsA[c], hbuf.data(), hsA[c],
                           infoA + c);
      nw[c] = q.ng;
    }
    return r == CUSOLVER_STATUS_SUCCESS ? std::string() : "cuSOLVER eigensolver failed in sector " + std::to_string(c);
  };
  auto jobA = [&](int l, int c, std::vector<char>& hbuf) -> std::string {
    std::string e = gram(l, c);
    return e.empty() ? eig(l, c, hbuf) : e;
  };
  std::vector<std::vector<double>> w(ns);
  auto fetch = [&](const std::vector<int>& secs) -> tn_status {
    std::vector<int> info(ns, 0);
    for (int c : secs) {
      w[c].resize(nw[c]);
      if (nw[c] == 0) continue;
      tn_status r = cuda_check(cudaMemcpyAsync(w[c].data(), A + oW[c], w[c].size() * 8, cudaMemcpyDeviceToHost, s), "D2H w");
      if (r != TN_OK) return r;
    }
    tn_status r = cuda_check(cudaMemcpyAsync(info.data(), infoA, ns * 4, cudaMemcpyDeviceToHost, s), "D2H info");
    if (r == TN_OK) r = cuda_check(cudaStreamSynchronize(s), "Gram sync");
    if (r != TN_OK) return r;
    for (int c : secs)
      if (info[c] != 0) return fail(TN_ERR_CUDA, "tn_svd_truncate: the eigensolver failed in sector " + std::to_string(c));
    return TN_OK;
  };
  const double eps = std::ldexp(1.0, -53);
  auto delta = [&](int c) { return w[c].empty() ? 0.0 : 16.0 * g[c].ng * eps * std::max(w[c].back(), 0.0); };
  // approximate χ-th largest s² over `secs` (−1 if fewer than χ values) and the largest error bound
  auto kth = [&](const std::vector<int>& secs, double& dmax) {
    std::vector<double> v;
    dmax = 0.0;
    for (int c : secs) {
      for (double x : w[c]) v.push_back(std::max(x, 0.0));
      dmax = std::max(dmax, delta(c));
    }
    if ((int64_t)v.size() < chi_max) return -1.0;
    std::nth_element(v.begin(), v.begin() + (chi_max - 1), v.end(), std::greater<double>());
    return v[chi_max - 1];
  };
  const bool prof = getenv("TN_SVD_PROFILE") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t0 = now();
  if ((st = run_lanes(X, s, wave1, cost, jobA)) != TN_OK) return st;
  if ((st = fetch(wave1)) != TN_OK) return st;
  const double t1 = now();
  double d1 = 0.0;
  const double T1 = kth(wave1, d1);
  // sectors at least this large get the trace-power test (TN_SVD_TEST_MIN_NG lets tests reach it at small sizes)
  const int test_min_ng = getenv("TN_SVD_TEST_MIN_NG") ? atoi(getenv("TN_SVD_TEST_MIN_NG")) : 256;
  std::vector<int> wave2, done(wave1), tested;
  // wave-2 sectors need only the eigenvalues that can still reach the exact top χ: T_final ≥ T1 (more sectors only
  // raise the χ-th value), and a sector's eigenvalue error is ≤ Δ_c ≤ 16·n_g·ε·‖Θ(c)‖²_F (its trace bounds λ_max)
  // Phase C keeps w ≥ max(τ, cutoff² − Δ_c) with τ = T2 − 2·max Δ ≥ T1 − 2D, D bounding every Δ; so vl = T1 − 2D
  // can never cut a value phase C would keep.
  if (T1 > 0.0) {
    double D = d1;
    for (int c : rest) D = std::max(D, 16.0 * g[c].ng * eps * n2[c]);
    const double vl = T1 - 2.0 * D;
    for (int c : rest) vlo[c] = vl > 0.0 ? vl : -1.0;
  }
  for (int c : rest) {
    if (T1 > 0.0 && n2[c] < T1 - d1) {
      disc_skipped += n2[c];
      sp.sec[c].k = 0;
    } else if (T1 - d1 > 0.0 && g[c].ng >= test_min_ng) {
      tested.push_back(c);
    } else {
      wave2.push_back(c);
    }
  }
  // Trace-power test for the remaining large sectors: with τ = T1 − d1 ≤ the exact χ-th s², every
  // eigenvalue λ ≥ τ of G contributes ≥ 1 to tr((G/τ)^16) = ‖(G/τ)^8‖²_F (three ZGEMM squarings), so a
  // sector with tr < 1/2 has no value that can enter the top χ and is skipped without its eigensolver
  // (an overflow or NaN fails the test, i.e. the sector is solved).
  if (!tested.empty()) {
    const double tau1 = T1 - d1;
    std::vector<size_t> oH(ns, 0);
    size_t hoff = 0;
    for (int c : tested) {
      oH[c] = hoff;
      hoff += (((size_t)g[c].ng * g[c].ng * 16 + 255) & ~(size_t)255) * 2;
    }
    char* Hb = nullptr;
    if ((st = grow(X.gbuf[2], X.gcap[2], hoff + 256 * (size_t)ns, &Hb)) != TN_OK) return st;
    double* d_tr = reinterpret_cast<double*>(Hb + hoff);
    const cuDoubleComplex inv2 = make_cuDoubleComplex(1.0 / (tau1 * tau1), 0.0);
    auto jobT = [&](int l, int c, std::vector<char>&) -> std::string {
      std::string e = gram(l, c);
      if (!e.empty()) return e;
      const int n = g[c].ng;
      const auto* G = reinterpret_cast<const cuDoubleComplex*>(A + oG[c]);
      auto* H1 = reinterpret_cast<cuDoubleComplex*>(Hb + oH[c]);
      auto* H2 = reinterpret_cast<cuDoubleComplex*>(Hb + oH[c] + (((size_t)n * n * 16 + 255) & ~(size_t)255));
      cublasStatus_t b = cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &inv2, G, n, G, n, &zero, H1, n);  // (G/τ)²
      if (b == CUBLAS_STATUS_SUCCESS)
        b = cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, H1, n, H1, n, &zero, H2, n);              // ^4
      if (b == CUBLAS_STATUS_SUCCESS)
        b = cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, H2, n, H2, n, &zero, H1, n);              // ^8
      return b == CUBLAS_STATUS_SUCCESS ? std::string() : "cuBLAS trace-power test failed in sector " + std::to_string(c);
    };
    if ((st = run_lanes(X, s, tested, cost, jobT)) != TN_OK) return st;
    ThetaPtrs tp{};
    for (int c : tested) {
      tp.p[c] = reinterpret_cast<const double2*>(Hb + oH[c]);
      tp.n[c] = (int64_t)g[c].ng * g[c].ng;
    }
    if ((st = cuda_check(cudaMemsetAsync(d_tr, 0, ns * sizeof(double), s), "memset tr")) != TN_OK) return st;
    k_sector_norm2<<<dim3(32, ns), 256, 0, s>>>(tp, d_tr);
    std::vector<double> tr(ns, 0.0);
    if ((st = cuda_check(cudaMemcpyAsync(tr.data(), d_tr, ns * 8, cudaMemcpyDeviceToHost, s), "D2H tr")) != TN_OK) return st;
    if ((st = cuda_check(cudaStreamSynchronize(s), "trace-power sync")) != TN_OK) return st;
    std::vector<int> solve;
    for (int c : tested) {
      if (tr[c] < 0.5) {
        disc_skipped += n2[c];
        sp.sec[c].k = 0;
      } else {
        solve.push_back(c);
      }
    }
    if (prof)
      for (int c : tested) fprintf(stderr, "[svd_gram]   trace-power test sector %d: tr((G/τ)^16) = %.3g\n", c, tr[c]);
    if ((st = run_lanes(X, s, solve, cost, eig)) != TN_OK) return st;
    if ((st = fetch(solve)) != TN_OK) return st;
    done.insert(done.end(), solve.begin(), solve.end());
  }
  if ((st = run_lanes(X, s, wave2, cost, jobA)) != TN_OK) return st;
  if ((st = fetch(wave2)) != TN_OK) return st;
  done.insert(done.end(), wave2.begin(), wave2.end());
  const double t2 = now();
  double dmax = 0.0;
  const double T2 = kth(done, dmax);
  const double tau = T2 > 0.0 ? T2 - 2.0 * dmax : -1.0;
  // phase C: k' per sector and its scratch
  std::vector<int> kp(ns, 0), waveC;
  std::vector<size_t> oT(ns), oP(ns), oWm(ns), oS(ns), oEW(ns), oWc(ns), wsC(ns), hsC(ns);
  std::vector<size_t> oM(ns), oV(ns), oW2(ns), oS2(ns), oSrc(ns), oRho(ns);   // Ritz refinement scratch
  off = 0;
  for (int c : done) {
    const double lo = std::max(tau, cutoff * cutoff - delta(c));
    int k = 0;
    for (int i = (int)nw[c] - 1; i >= 0 && w[c][i] >= lo; --i) ++k;
    kp[c] = k;
    if (k == 0) {
      disc_skipped += n2[c];
      sp.sec[c].k = 0;
      continue;
    }
    waveC.push_back(c);
    const Geo& q = g[c];
    if (cusolverDnXgesvdp_bufferSize(X.h[0], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, q.mt, k, CUDA_C_64F, nullptr, q.mt,
                                     CUDA_R_64F, nullptr, CUDA_C_64F, nullptr, q.mt, CUDA_C_64F, nullptr, k, CUDA_C_64F,
                                     &wsC[c], &hsC[c]) != CUSOLVER_STATUS_SUCCESS)
      return fail(TN_ERR_CUDA, "cusolverDnXgesvdp_bufferSize failed");
    oT[c] = take((size_t)q.mt * k * 16);
    oP[c] = take((size_t)q.mt * k * 16);
    oWm[c] = take((size_t)k * k * 16);
    oS[c] = take((size_t)k * 8);
    oEW[c] = take((size_t)q.ng * k * 16);
    oWc[c] = take(wsC[c]);
    oM[c] = take((size_t)k * k * 16);
    oV[c] = take((size_t)k * k * 16);
    oW2[c] = take((size_t)k * k * 16);
    oS2[c] = take((size_t)k * 8);
    oSrc[c] = take((size_t)k * 4);
    oRho[c] = take(8);
  }
  char* Cb = nullptr;
  if ((st = grow(X.gbuf[1], X.gcap[1], std::max<size_t>(off, 256), &Cb)) != TN_OK) return st;
  std::atomic<int> n_jacobi{0}, n_refined{0}, n_refine_fallback{0}, n_passes{0};
  // Ritz refinement (k_ritz_rot above): 0 = done (P, Wm, S written), 1 = did not converge (caller falls back to a
  // library SVD of a recomputed Y), -1 = a CUDA / cuBLAS error
  auto refine = [&](int l, int c, int mt, int k, double2* T, std::string& err) -> int {
    cublasHandle_t hb = X.hb[l];
    cudaStream_t st = X.st[l];
    double2* Ya = T;
    double2* Yb = reinterpret_cast<double2*>(Cb + oP[c]);
    double2* Wa = reinterpret_cast<double2*>(Cb + oWm[c]);
    double2* Wb = reinterpret_cast<double2*>(Cb + oW2[c]);
    double2* M = reinterpret_cast<double2*>(Cb + oM[c]);
    double2* V = reinterpret_cast<double2*>(Cb + oV[c]);
    auto* rho_d = reinterpret_cast<unsigned long long*>(Cb + oRho[c]);
    auto cz = [](double2* p) { return reinterpret_cast<cuDoubleComplex*>(p); };
    const unsigned gk = (unsigned)std::min<int64_t>(1024, ((int64_t)k * k + 255) / 256);
    auto gemm = [&](cublasOperation_t ta, int mm, int nn, int kk, const double2* A_, int lda, const double2* B_, int ldb,
                    double2* C_, int ldc) {
      return cublasZgemm(hb, ta, CUBLAS_OP_N, mm, nn, kk, &one, reinterpret_cast<const cuDoubleComplex*>(A_), lda,
                         reinterpret_cast<const cuDoubleComplex*>(B_), ldb, &zero, cz(C_), ldc) == CUBLAS_STATUS_SUCCESS;
    };
    // ρ_max of Y's column pairs (M = YᴴY, V = the simultaneous rotation); the one host sync per pass
    auto measure = [&](double& rho) -> bool {
      if (!gemm(CUBLAS_OP_C, k, k, mt, Ya, mt, Ya, mt, M, k)) return false;
      if (cudaMemsetAsync(rho_d, 0, 8, st) != cudaSuccess) return false;
      k_ritz_rot<<<gk, 256, 0, st>>>(M, k, V, rho_d);
      unsigned long long bits = 0;
      if (cudaMemcpyAsync(&bits, rho_d, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) return false;
      if (cudaStreamSynchronize(st) != cudaSuccess) return false;
      rho = __builtin_bit_cast(double, bits);
      return true;
    };
    // converged when every column pair is orthogonal to rounding of the dot products that measure it
    const double tol = 16.0 * std::sqrt((double)mt) * std::ldexp(1.0, -53);
    k_eye<<<gk, 256, 0, st>>>(Wa, k, 1.0, 0.0);
    bool conv = false, applied = false;
    double rho = 0.0;
    const bool prof_r = prof;
    for (int pass = 0; pass < 8; ++pass) {
      if (!measure(rho)) return err = "Ritz refinement (measure) failed in sector " + std::to_string(c), -1;
      ++n_passes;
      if (prof_r) fprintf(stderr, "[svd] refine sector %d %dx%d pass %d rho %.3e\n", c, mt, k, pass, rho);
      if (rho <= tol) {
        conv = true;
        break;
      }
      if (!(rho < 0.5)) break;  // far from orthogonal (clusters, noise-level columns): leave it to the library SVD
      if (!gemm(CUBLAS_OP_N, mt, k, k, Ya, mt, V, k, Yb, mt) || !gemm(CUBLAS_OP_N, k, k, k, Wa, k, V, k, Wb, k))
        return err = "Ritz refinement (rotate) failed in sector " + std::to_string(c), -1;
      std::swap(Ya, Yb);
      std::swap(Wa, Wb);
      applied = true;
    }
    if (!conv) return 1;
    if (applied) {
      // one Newton–Schulz step makes the accumulated rotation unitary to rounding: C = (3I − WᴴW)/2,
      // W ← W·C, Y ← Y·C; then the pairs are measured once more
      if (!gemm(CUBLAS_OP_C, k, k, k, Wa, k, Wa, k, M, k)) return err = "Ritz refinement (NS) failed", -1;
      k_eye<<<gk, 256, 0, st>>>(M, k, 1.5, -0.5);
      if (!gemm(CUBLAS_OP_N, mt, k, k, Ya, mt, M, k, Yb, mt) || !gemm(CUBLAS_OP_N, k, k, k, Wa, k, M, k, Wb, k))
        return err = "Ritz refinement (NS) failed", -1;
      std::swap(Ya, Yb);
      std::swap(Wa, Wb);
      if (!measure(rho)) return err = "Ritz refinement (check) failed in sector " + std::to_string(c), -1;
      if (rho > tol) return 1;
    }
    // outputs P (Cb + oP), Wm (Cb + oWm), S: stage the current Y / W out of the output buffers first
    double2* Pout = reinterpret_cast<double2*>(Cb + oP[c]);
    double2* Wout = reinterpret_cast<double2*>(Cb + oWm[c]);
    if (Ya == Pout) {
      if (cudaMemcpyAsync(T, Ya, (size_t)mt * k * 16, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return err = "Ritz refinement copy failed", -1;
      Ya = T;
    }
    if (Wa == Wout) {
      if (cudaMemcpyAsync(Wb, Wa, (size_t)k * k * 16, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return err = "Ritz refinement copy failed", -1;
      Wa = Wb;
    }
    auto* s2 = reinterpret_cast<double*>(Cb + oS2[c]);
    auto* src = reinterpret_cast<int32_t*>(Cb + oSrc[c]);
    k_colnorm2<<<k, 256, 0, st>>>(Ya, mt, s2);
    k_ritz_rank<<<(k + 255) / 256, 256, 0, st>>>(s2, k, src);
    const int64_t tot = (int64_t)mt * k + (int64_t)k * k + k;
    k_ritz_permute<<<(unsigned)std::min<int64_t>(4096, (tot + 255) / 256), 256, 0, st>>>(
        Ya, Wa, s2, src, mt, k, Pout, Wout, reinterpret_cast<double*>(Cb + oS[c]));
    if (cudaGetLastError() != cudaSuccess) return err = "Ritz refinement kernels failed", -1;
    ++n_refined;
    return 0;
  };
  auto jobC = [&](int l, int c, std::vector<char>& hbuf) -> std::string {
    const Geo& q = g[c];
    const int k = kp[c];
    const auto* Z = reinterpret_cast<const cuDoubleComplex*>(theta[c]);
    const auto* E = reinterpret_cast<const cuDoubleComplex*>(A + oG[c]) + (size_t)(nw[c] - k) * q.ng;
    auto* T = reinterpret_cast<cuDoubleComplex*>(Cb + oT[c]);
    auto* Wm = reinterpret_cast<cuDoubleComplex*>(Cb + oWm[c]);
    cublasStatus_t b =
        q.tall ? cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, q.C, k, q.R, &one, Z, q.C, E, q.R, &zero, T, q.C)
               : cublasZgemm(X.hb[l], CUBLAS_OP_C, CUBLAS_OP_N, q.R, k, q.C, &one, Z, q.C, E, q.C, &zero, T, q.R);
    if (b != CUBLAS_STATUS_SUCCESS) return "cuBLAS Ritz projection failed in sector " + std::to_string(c);
    // default: the Ritz refinement above (GEMMs + own kernels; Y's columns are already nearly orthogonal);
    // TN_RITZ_SVD=1 (or a refinement that does not converge) takes a library SVD of Y instead: one-sided Jacobi
    // for narrow Y (config 3: 89 ms for the Ritz phase vs 110 ms with the polar-decomposition Xgesvdp, which
    // TN_RITZ_POLAR=1 selects, guarded by its backward-error report)
    const bool force_polar = getenv("TN_RITZ_POLAR") != nullptr;
    const bool library_ritz = force_polar || getenv("TN_RITZ_SVD") != nullptr;
    bool refine_failed = false;
    if (!library_ritz) {
      std::string err;
      const int r = refine(l, c, q.mt, k, reinterpret_cast<double2*>(T), err);
      if (r < 0) return err;
      if (r == 0) {
        b = cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, q.ng, k, k, &one, E, q.ng, Wm, k, &zero,
                        reinterpret_cast<cuDoubleComplex*>(Cb + oEW[c]), q.ng);
        return b == CUBLAS_STATUS_SUCCESS ? std::string() : "cuBLAS Ritz rotation failed in sector " + std::to_string(c);
      }
      ++n_refine_fallback;
      refine_failed = true;
    }
    // Jacobi for narrow Y; for wide ones (k' > 512: wide spectra where the Gram bound keeps most values, e.g.
    // MPO gates) the GEMM-rich polar decomposition is faster (MPO pair-config-3 layer: 4.9 → 5.9 gates/s)
    const bool ritz_jacobi = !force_polar && k <= 512;
    (void)refine_failed;
    double herr = 0.0;
    if (!ritz_jacobi) {
      hbuf.resize(std::max<size_t>(hsC[c], 1));
      const cusolverStatus_t r =
          cusolverDnXgesvdp(X.h[l], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, q.mt, k, CUDA_C_64F, T, q.mt, CUDA_R_64F,
                            Cb + oS[c], CUDA_C_64F, Cb + oP[c], q.mt, CUDA_C_64F, Wm, k, CUDA_C_64F, Cb + oWc[c], wsC[c],
                            hbuf.data(), hsC[c], infoC + c, &herr);
      if (r != CUSOLVER_STATUS_SUCCESS) return "cuSOLVER Ritz SVD failed in sector " + std::to_string(c);
      if (getenv("TN_SVD_PROFILE")) fprintf(stderr, "[svd] ritz sector %d %dx%d h_err_sigma %.3e\n", c, q.mt, k, herr);
    }
    if (ritz_jacobi || !(herr <= kRitzHerrMax)) {
      // the polar-decomposition SVD reports a large backward error (seen up to 5e-8 on small rank-deficient
      // matrices): recompute Y and take the one-sided Jacobi SVD instead (accurate to rounding, slower)
      ++n_jacobi;
      b = q.tall ? cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, q.C, k, q.R, &one, Z, q.C, E, q.R, &zero, T, q.C)
                 : cublasZgemm(X.hb[l], CUBLAS_OP_C, CUBLAS_OP_N, q.R, k, q.C, &one, Z, q.C, E, q.C, &zero, T, q.R);
      if (b != CUBLAS_STATUS_SUCCESS) return "cuBLAS Ritz projection failed in sector " + std::to_string(c);
      gesvdjInfo_t jp = nullptr;
      if (cusolverDnCreateGesvdjInfo(&jp) != CUSOLVER_STATUS_SUCCESS) return "cusolverDnCreateGesvdjInfo failed";
      cusolverDnXgesvdjSetTolerance(jp, 0.0);
      cusolverDnXgesvdjSetMaxSweeps(jp, 100);
      int lw = 0;
      std::string err;
      if (cusolverDnZgesvdj_bufferSize(X.h[l], CUSOLVER_EIG_MODE_VECTOR, 1, q.mt, k, T, q.mt,
                                       reinterpret_cast<double*>(Cb + oS[c]), reinterpret_cast<cuDoubleComplex*>(Cb + oP[c]),
                                       q.mt, Wm, k, &lw, jp) != CUSOLVER_STATUS_SUCCESS) {
        err = "cusolverDnZgesvdj_bufferSize failed";
      } else {
        void* wj = nullptr;
        if (cudaMallocAsync(&wj, (size_t)std::max(lw, 1) * 16, X.st[l]) != cudaSuccess) {
          err = "Jacobi workspace allocation failed";
        } else {
          if (cusolverDnZgesvdj(X.h[l], CUSOLVER_EIG_MODE_VECTOR, 1, q.mt, k, T, q.mt,
                                reinterpret_cast<double*>(Cb + oS[c]), reinterpret_cast<cuDoubleComplex*>(Cb + oP[c]),
                                q.mt, Wm, k, reinterpret_cast<cuDoubleComplex*>(wj), lw, infoC + c, jp) !=
              CUSOLVER_STATUS_SUCCESS)
            err = "cuSOLVER Jacobi Ritz SVD failed in sector " + std::to_string(c);
          cudaFreeAsync(wj, X.st[l]);
        }
      }
      cusolverDnDestroyGesvdjInfo(jp);
      if (!err.empty()) return err;
    }
    b = cublasZgemm(X.hb[l], CUBLAS_OP_N, CUBLAS_OP_N, q.ng, k, k, &one, E, q.ng, Wm, k, &zero,
                    reinterpret_cast<cuDoubleComplex*>(Cb + oEW[c]), q.ng);
    return b == CUBLAS_STATUS_SUCCESS ? std::string() : "cuBLAS Ritz rotation failed in sector " + std::to_string(c);
  };
  if ((st = run_lanes(X, s, waveC, cost, jobC)) != TN_OK) return st;
  if (prof)
    fprintf(stderr, "[svd_gram] Ritz: %d refined (%d passes), %d refinement fallbacks, %d Jacobi SVDs\n",
            n_refined.load(), n_passes.load(), n_refine_fallback.load(), n_jacobi.load());
  std::vector<int> info(ns, 0);
  std::vector<std::vector<double>> sv(ns);
  for (int c : waveC) {
    sv[c].resize(kp[c]);
    if ((st = cuda_check(cudaMemcpyAsync(sv[c].data(), Cb + oS[c], kp[c] * 8, cudaMemcpyDeviceToHost, s), "D2H S")) != TN_OK)
      return st;
  }
  if ((st = cuda_check(cudaMemcpyAsync(info.data(), infoC, ns * 4, cudaMemcpyDeviceToHost, s), "D2H info")) != TN_OK)
    return st;
  if ((st = cuda_check(cudaStreamSynchronize(s), "Ritz sync")) != TN_OK) return st;
  if (prof) {
    int64_t sk = 0, sn = 0;
    int kmax = 0;
    for (int c : waveC) {
      sk += kp[c];
      sn += g[c].ng;
      kmax = std::max(kmax, kp[c]);
    }
    fprintf(stderr, "[svd_gram] gram+eig wave1 %.1f ms (%zu sectors), wave2 %.1f ms (%zu), ritz %.1f ms (%zu sectors, sum k' %lld of %lld, max k' %d)\n",
            t1 - t0, wave1.size(), t2 - t1, wave2.size(), now() - t2, waveC.size(), (long long)sk, (long long)sn, kmax);
    for (int c : done)
      fprintf(stderr, "[svd_gram]   sector %d: %dx%d n_g %d k' %d  |Θ|²/T² %.1f  wave %d\n", c, g[c].R, g[c].C, g[c].ng,
              kp[c], T2 > 0 ? n2[c] / T2 : -1.0,
              std::find(wave1.begin(), wave1.end(), c) != wave1.end() ? 1 : 2);
  }
  for (int c : waveC) {
    if (info[c] != 0) return fail(TN_ERR_CUDA, "tn_svd_truncate: the Ritz SVD failed in sector " + std::to_string(c));
    if (kp[c] < g[c].ng) {  // the weight outside the computed values (none when all n_g were computed)
      double kept2 = 0.0;
      for (double x : sv[c]) kept2 += x * x;
      disc_skipped += std::max(n2[c] - kept2, 0.0);
    }
    SvdSector& S = sp.sec[c];
    const double2* P = reinterpret_cast<const double2*>(Cb + oP[c]);
    const double2* EW = reinterpret_cast<const double2*>(Cb + oEW[c]);
    S.ux = g[c].tall ? P : EW;   // C × k', ld C
    S.vx = g[c].tall ? EW : P;   // R × k', ld R
    S.s = reinterpret_cast<const double*>(Cb + oS[c]);
    S.k = kp[c];
  }
  return TN_OK;
}

}  // namespace tn

using namespace tn;

// form 0: Vidal factors (tn_svd_truncate); form 1: right-canonical factors (tn_svd_truncate_bform)
static tn_status svd_truncate_impl(const tn_plan* p, tn_stream stream, double* const* theta, const double* lambda_l,
                                   const double* lambda_r, int64_t chi_max, double cutoff, int32_t* q_new,
                                   double* lambda_new, double* gamma_k_new, double* gamma_k1_new, int64_t* chi_out,
                                   double* discarded, int form) {
  if (chi_max < 1 || !(cutoff >= 0.0)) return fail(TN_ERR_DOMAIN, "tn_svd_truncate: chi_max < 1 or cutoff < 0");
  if (!p || !theta || !lambda_l || (!lambda_r && form == 0) || !q_new || !lambda_new || !gamma_k_new ||
      !gamma_k1_new || !chi_out || !discarded)
    return fail(TN_ERR_DIMENSION, "tn_svd_truncate: NULL argument");
  if (p->world != 1) return fail(TN_ERR_UNSUPPORTED, "tn_svd_truncate: needs a single-GPU plan (full sectors)");
  if (p->nsec > SVD_MAXSEC) return fail(TN_ERR_UNSUPPORTED, "tn_svd_truncate: more sectors than this build's SVD step handles");
  cudaStream_t s = (cudaStream_t)stream;
  if (tn_status w = wait_tables(p, s); w != TN_OK) return w;   // the factors read the plan's perm tables
  SvdCtx& X = ctx();
  std::lock_guard<std::mutex> lock(X.mu);
  if (!X.h[0]) {
    for (int i = 0; i < SVD_LANES; ++i) {
      if (cusolverDnCreate(&X.h[i]) != CUSOLVER_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "cusolverDnCreate failed");
      if (cudaStreamCreateWithFlags(&X.st[i], cudaStreamNonBlocking) != cudaSuccess)
        return fail(TN_ERR_CUDA, "SVD stream create failed");
      cusolverDnSetStream(X.h[i], X.st[i]);
      if (cublasCreate(&X.hb[i]) != CUBLAS_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "cublasCreate failed");
      cublasSetStream(X.hb[i], X.st[i]);
    }
    for (auto& e : X.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return fail(TN_ERR_CUDA, "event");
    if (cusolverDnCreateGesvdjInfo(&X.params) != CUSOLVER_STATUS_SUCCESS)
      return fail(TN_ERR_CUDA, "cusolverDnCreateGesvdjInfo failed");
    cusolverDnXgesvdjSetTolerance(X.params, 0.0);      // 0 → machine accuracy
    cusolverDnXgesvdjSetMaxSweeps(X.params, 100);
    for (auto& q : X.pj) {
      if (cusolverDnCreateGesvdjInfo(&q) != CUSOLVER_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "gesvdj info");
      cusolverDnXgesvdjSetTolerance(q, 0.0);
      cusolverDnXgesvdjSetMaxSweeps(q, 100);
    }
    if (cusolverDnCreateParams(&X.xparams) != CUSOLVER_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "cusolver params");
  }
  const int algo = svd_algo();
  const int ns = p->nsec;
  // ---- scratch layout: per sector U_x, V_x, S, workspace (library SVD paths); then sort buffers ----
  SvdParams sp{};
  sp.nsec = ns;
  std::vector<size_t> o_ux(ns), o_vx(ns), o_s(ns), o_w(ns);
  std::vector<int> lwork(ns, 0);
  std::vector<size_t> hbytes(ns, 0), wsz(ns, 0);
  std::vector<int64_t> base(ns + 1, 0);
  size_t off = 0, copy_max = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  for (int c = 0; c < ns; ++c) {
    const int R = (int)p->R[c], C = (int)p->C[c], k = std::min(R, C);
    base[c + 1] = base[c] + k;
    if (k == 0 || algo == 2) continue;
    size_t wbytes = 0;
    // Jacobi workspace: the gesvdj path, and the gesvdp path's fallback
    if (cusolverDnZgesvdj_bufferSize(X.h[0], CUSOLVER_EIG_MODE_VECTOR, 1, C, R, nullptr, C, nullptr, nullptr, C,
                                     nullptr, R, &lwork[c], X.params) != CUSOLVER_STATUS_SUCCESS)
      return fail(TN_ERR_CUDA, "cusolverDnZgesvdj_bufferSize failed");
    copy_max = std::max(copy_max, (size_t)R * C * 16);
    if (algo == 0) {
      wbytes = (size_t)lwork[c] * 16;
    } else {
      size_t hb = 0;
      if (cusolverDnXgesvdp_bufferSize(X.h[0], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, C, R, CUDA_C_64F, nullptr, C,
                                       CUDA_R_64F, nullptr, CUDA_C_64F, nullptr, C, CUDA_C_64F, nullptr, R, CUDA_C_64F,
                                       &wbytes, &hb) != CUSOLVER_STATUS_SUCCESS)
        return fail(TN_ERR_CUDA, "cusolverDnXgesvdp_bufferSize failed");
      hbytes[c] = hb;
      wbytes = std::max(wbytes, (size_t)lwork[c] * 16);
    }
    o_ux[c] = take((size_t)C * k * 16);
    o_vx[c] = take((size_t)R * k * 16);
    o_s[c] = take((size_t)k * 8);
    o_w[c] = take(wbytes);
    wsz[c] = wbytes;
  }
  const int64_t total_max = base[ns];
  // library paths: each lane factorises a copy of Θ(c) (the routines overwrite their input; Θ stays intact)
  const size_t o_copy = take(copy_max * SVD_LANES);
  const size_t o_info = take((size_t)ns * 4);
  const size_t o_n2 = take((size_t)ns * 8);
  const size_t o_kin = take((size_t)std::max<int64_t>(total_max, 1) * 8),
               o_kout = take((size_t)std::max<int64_t>(total_max, 1) * 8);
  const size_t o_vin = take((size_t)std::max<int64_t>(total_max, 1) * 4),
               o_vout = take((size_t)std::max<int64_t>(total_max, 1) * 4);
  const size_t o_base = take((size_t)(ns + 1) * 8);
  const size_t o_off = take((size_t)(ns + 1) * 4);
  const size_t o_res = take(16);
  // pair plans: Θ(c1,c2)'s rows are whole left pair segments (l1 ∈ [c1, c1+d−1], l2 ∈ [c2, c2+d−1], key order)
  // and its columns whole right segments (r1 ∈ [c1−d+1, c1], r2 ∈ [c2−d+1, c2]) — tn_pair.cu's layout
  std::vector<int32_t> hpos;
  std::vector<int64_t> rpos_at(ns, 0), cpos_at(ns, 0);
  if (p->pair) {
    const int N = p->N, d = p->d, nk = N + 1;
    const auto& ol = p->off[0];
    const auto& orr = p->off[2];
    for (int c = 0; c < ns; ++c) {
      const int c1 = c / nk, c2 = c % nk;
      rpos_at[c] = (int64_t)hpos.size();
      for (int l1 = c1; l1 <= std::min(N, c1 + d - 1); ++l1)
        for (int l2 = c2; l2 <= std::min(N, c2 + d - 1); ++l2)
          for (int32_t x = ol[l1 * nk + l2]; x < ol[l1 * nk + l2 + 1]; ++x) hpos.push_back(x);
      if ((int64_t)hpos.size() - rpos_at[c] != p->R[c]) return fail(TN_ERR_CONSISTENCY, "tn_svd_truncate: pair rows");
      cpos_at[c] = (int64_t)hpos.size();
      for (int r1 = std::max(0, c1 - d + 1); r1 <= c1; ++r1)
        for (int r2 = std::max(0, c2 - d + 1); r2 <= c2; ++r2)
          for (int32_t x = orr[r1 * nk + r2]; x < orr[r1 * nk + r2 + 1]; ++x) hpos.push_back(x);
      if ((int64_t)hpos.size() - cpos_at[c] != p->C[c]) return fail(TN_ERR_CONSISTENCY, "tn_svd_truncate: pair cols");
    }
  }
  const size_t o_pos = take(std::max<size_t>(hpos.size(), 1) * 4);
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const double*)nullptr, (double*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(total_max, 1));
  const size_t o_sort = take(sort_bytes);
  char* B = nullptr;
  tn_status st = grow(X.buf, X.cap, off, &B);
  if (st != TN_OK) return st;
  int* d_info = reinterpret_cast<int*>(B + o_info);
  std::vector<int> order;
  for (int c = 0; c < ns; ++c) {
    const int R = (int)p->R[c], C = (int)p->C[c], k = std::min(R, C);
    SvdSector& S = sp.sec[c];
    S.R = R;
    S.C = C;
    S.k = k;
    S.row0 = p->row0[c];
    S.col0 = p->col0[c];
    S.rpos = p->pair ? reinterpret_cast<const int32_t*>(B + o_pos) + rpos_at[c] : nullptr;
    S.cpos = p->pair ? reinterpret_cast<const int32_t*>(B + o_pos) + cpos_at[c] : nullptr;
    if (k == 0) continue;
    if (!theta[c]) return fail(TN_ERR_DIMENSION, "tn_svd_truncate: NULL Θ(c) for a non-empty sector");
    if (algo != 2) {
      S.ux = reinterpret_cast<double2*>(B + o_ux[c]);
      S.vx = reinterpret_cast<double2*>(B + o_vx[c]);
      S.s = reinterpret_cast<double*>(B + o_s[c]);
    }
    order.push_back(c);
  }
  st = cuda_check(cudaMemsetAsync(d_info, 0, ns * sizeof(int), s), "memset info");  // empty sectors
  if (st != TN_OK) return st;
  if (!hpos.empty() &&
      (st = cuda_check(cudaMemcpyAsync(B + o_pos, hpos.data(), hpos.size() * 4, cudaMemcpyHostToDevice, s),
                       "H2D pair positions")) != TN_OK)
    return st;
  auto cost = [&](int c) { return (double)p->R[c] * p->C[c] * std::min(p->R[c], p->C[c]); };
  // one library SVD (paths 0/1) of a lane-private copy of Θ(c): X = Θᵀ (column-major C × R, ld C) = U_x S V_xᴴ.
  // Xgesvdp (path 1) reports its backward error; above kLibHerrMax the sector is redone by Jacobi (seen:
  // 5e-8 on small rank-deficient sectors), so both paths are accurate to rounding
  auto lib_svd = [&](int l, int c, std::vector<char>& hbuf) -> std::string {
    const SvdSector& S = sp.sec[c];
    const int R = S.R, C = S.C;
    auto* Zc = reinterpret_cast<cuDoubleComplex*>(B + o_copy + (size_t)l * copy_max);
    auto copy_in = [&] {
      return cudaMemcpyAsync(Zc, theta[c], (size_t)R * C * 16, cudaMemcpyDeviceToDevice, X.st[l]) == cudaSuccess;
    };
    auto jacobi = [&] {
      return cusolverDnZgesvdj(X.h[l], CUSOLVER_EIG_MODE_VECTOR, 1, C, R, Zc, C, const_cast<double*>(S.s),
                               reinterpret_cast<cuDoubleComplex*>(const_cast<double2*>(S.ux)), C,
                               reinterpret_cast<cuDoubleComplex*>(const_cast<double2*>(S.vx)), R,
                               reinterpret_cast<cuDoubleComplex*>(B + o_w[c]), lwork[c], d_info + c, X.pj[l]);
    };
    if (!copy_in()) return "copy of sector " + std::to_string(c) + " failed";
    cusolverStatus_t r;
    if (algo == 0) {
      r = jacobi();
    } else {
      hbuf.resize(std::max<size_t>(hbytes[c], 1));
      double herr = 0.0;
      r = cusolverDnXgesvdp(X.h[l], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, C, R, CUDA_C_64F, Zc, C, CUDA_R_64F,
                            const_cast<double*>(S.s), CUDA_C_64F, const_cast<double2*>(S.ux), C, CUDA_C_64F,
                            const_cast<double2*>(S.vx), R, CUDA_C_64F, B + o_w[c], wsz[c], hbuf.data(), hbytes[c],
                            d_info + c, &herr);
      if (getenv("TN_SVD_PROFILE")) fprintf(stderr, "[svd] gesvdp sector %d %dx%d h_err_sigma %.3e\n", c, R, C, herr);
      if (r == CUSOLVER_STATUS_SUCCESS && !(herr <= kRitzHerrMax)) {
        if (!copy_in()) return "copy of sector " + std::to_string(c) + " failed";
        r = jacobi();
      }
    }
    return r == CUSOLVER_STATUS_SUCCESS ? std::string()
                                        : "cuSOLVER SVD failed in sector " + std::to_string(c) + " (status " +
                                              std::to_string((int)r) + ")";
  };
  // ---- norm bound: the largest singular value of Θ(c) is ≤ ‖Θ(c)‖_F, so a sector whose norm is below the
  // χ-th largest value found among the heaviest sectors cannot place any value in the global top χ (that
  // threshold only grows): its SVD is skipped and its whole weight ‖Θ(c)‖²_F is discarded ----
  double disc_skipped = 0.0;
  std::vector<double> n2(ns, 0.0);
  {
    ThetaPtrs tp{};
    for (int c = 0; c < ns; ++c) {
      tp.p[c] = reinterpret_cast<const double2*>(theta[c]);
      tp.n[c] = sp.sec[c].k ? (int64_t)p->R[c] * p->C[c] : 0;
    }
    double* d_n2 = reinterpret_cast<double*>(B + o_n2);
    if ((st = cuda_check(cudaMemsetAsync(d_n2, 0, ns * sizeof(double), s), "memset norms")) != TN_OK) return st;
    k_sector_norm2<<<dim3(32, ns), 256, 0, s>>>(tp, d_n2);
    if ((st = cuda_check(cudaMemcpyAsync(n2.data(), d_n2, ns * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H norms")) !=
        TN_OK)
      return st;
    if ((st = cuda_check(cudaStreamSynchronize(s), "norm sync")) != TN_OK) return st;
  }
  std::sort(order.begin(), order.end(), [&](int a, int b) { return n2[a] > n2[b]; });
  std::vector<int> wave1, rest;
  {
    // wave 1 = the heaviest sectors until they hold ≥ 3χ values: a larger first wave gives a higher χ-th value
    // and more skipped sectors, a smaller one solves fewer sectors blind (config 3: factor 2 / 2.5 / 3 / 3.5 /
    // 4 / 6 → 354 / 322 / 313 / 342 / 366 / 466 ms); TN_SVD_WAVE1 overrides
    static const double wave1_factor = getenv("TN_SVD_WAVE1") ? atof(getenv("TN_SVD_WAVE1")) : 3.0;
    int64_t have = 0;
    for (int c : order) {
      if (have < wave1_factor * chi_max) {
        wave1.push_back(c);
        have += sp.sec[c].k;
      } else {
        rest.push_back(c);
      }
    }
  }
  if (algo == 2) {
    if ((st = svd_gram(X, s, theta, sp, n2, wave1, rest, chi_max, cutoff, disc_skipped)) != TN_OK) return st;
  } else {
    if ((st = run_lanes(X, s, wave1, cost, lib_svd)) != TN_OK) return st;
    std::vector<int> wave2;
    if (!rest.empty()) {
      // the chi_max-th largest value of wave 1 (values of each sector come back descending)
      std::vector<double> vals;
      for (int c : wave1) {
        std::vector<double> v(sp.sec[c].k);
        if ((st = cuda_check(cudaMemcpyAsync(v.data(), sp.sec[c].s, v.size() * 8, cudaMemcpyDeviceToHost, s),
                             "D2H wave-1 values")) != TN_OK)
          return st;
        if ((st = cuda_check(cudaStreamSynchronize(s), "wave-1 sync")) != TN_OK) return st;
        vals.insert(vals.end(), v.begin(), v.end());
      }
      double T = -1.0;
      if ((int64_t)vals.size() >= chi_max) {
        std::nth_element(vals.begin(), vals.begin() + (chi_max - 1), vals.end(), std::greater<double>());
        T = vals[chi_max - 1];
      }
      for (int c : rest) {
        if (T > 0.0 && std::sqrt(n2[c]) < T) {
          disc_skipped += n2[c];
          sp.sec[c].k = 0;  // skipped: contributes no value, its whole weight is discarded
        } else {
          wave2.push_back(c);
        }
      }
      if ((st = run_lanes(X, s, wave2, cost, lib_svd)) != TN_OK) return st;
    }
  }
  for (int c = 0; c < ns; ++c) base[c + 1] = base[c] + sp.sec[c].k;
  const int64_t total = base[ns];
  double* kin = reinterpret_cast<double*>(B + o_kin);
  double* kout = reinterpret_cast<double*>(B + o_kout);
  int32_t* vin = reinterpret_cast<int32_t*>(B + o_vin);
  int32_t* vout = reinterpret_cast<int32_t*>(B + o_vout);
  int64_t* d_base = reinterpret_cast<int64_t*>(B + o_base);
  int32_t* d_off = reinterpret_cast<int32_t*>(B + o_off);
  int64_t* d_chi = reinterpret_cast<int64_t*>(B + o_res);
  double* d_disc = reinterpret_cast<double*>(B + o_res + 8);
  st = cuda_check(cudaMemcpyAsync(d_base, base.data(), (ns + 1) * 8, cudaMemcpyHostToDevice, s), "H2D bases");  // after skips
  if (st != TN_OK) return st;
  if (total > 0) {
    k_svd_pack<<<dim3(8, ns), 256, 0, s>>>(sp, kin, vin, d_base);
    size_t sb = sort_bytes;
    if (cub::DeviceRadixSort::SortPairsDescending(B + o_sort, sb, kin, kout, vin, vout, (int)total, 0, 64, s) !=
        cudaSuccess)
      return fail(TN_ERR_CUDA, "radix sort of singular values failed");
  }
  k_svd_select<<<1, 1024, 0, s>>>(sp, kout, vout, total, chi_max, cutoff, q_new, lambda_new, d_off, d_chi, d_disc,
                                  disc_skipped);
  if ((st = cuda_check(cudaGetLastError(), "SVD select")) != TN_OK) return st;
  std::vector<int> info(ns, 0);
  int64_t res[2];
  if ((st = cuda_check(cudaMemcpyAsync(info.data(), d_info, ns * 4, cudaMemcpyDeviceToHost, s), "D2H info")) != TN_OK)
    return st;
  if ((st = cuda_check(cudaMemcpyAsync(res, d_chi, 16, cudaMemcpyDeviceToHost, s), "D2H results")) != TN_OK) return st;
  if ((st = cuda_check(cudaStreamSynchronize(s), "SVD sync")) != TN_OK) return st;
  for (int c = 0; c < ns; ++c)
    if (info[c] != 0)
      return fail(TN_ERR_CUDA, "tn_svd_truncate: the SVD failed in sector " + std::to_string(c) + " (" +
                                   std::to_string(p->R[c]) + "x" + std::to_string(p->C[c]) + ", info " +
                                   std::to_string(info[c]) + ")");
  // factors in their compact layout: Γk_new [χ_l × χ_new] (ld χ_new), Γk1_new [χ_new × χ_r]
  const int64_t chi_new = res[0];
  if (chi_new > 0) {
    if ((st = cuda_check(cudaMemsetAsync(gamma_k_new, 0, (size_t)p->chi[0] * chi_new * 16, s), "memset Γk_new")) != TN_OK)
      return st;
    if ((st = cuda_check(cudaMemsetAsync(gamma_k1_new, 0, (size_t)chi_new * p->chi[2] * 16, s), "memset Γk1_new")) !=
        TN_OK)
      return st;
    if (form == 0) {
      k_svd_factors<<<dim3(std::max(1, 2 * p->sm_count / std::max(1, ns) + 1), ns), 256, 0, s>>>(
          sp, d_off, p->d_perm[0], p->d_perm[2], lambda_l, lambda_r, chi_new, p->chi[2],
          reinterpret_cast<double2*>(gamma_k_new), reinterpret_cast<double2*>(gamma_k1_new));
      if ((st = cuda_check(cudaGetLastError(), "SVD factors")) != TN_OK) return st;
    } else {
      // right-canonical form (R22): B^{[k]}_new = Θ(c)·V_c / λl (one ZGEMM per sector, T = U_xᴴ·Z with
      // Z = Θ(c)ᵀ column-major, then a scatter that undoes Θ's row scaling), B^{[k+1]}_new = V_c† = U_xᵀ
      std::vector<int32_t> hoff(ns + 1, 0);
      if ((st = cuda_check(cudaMemcpyAsync(hoff.data(), d_off, (ns + 1) * 4, cudaMemcpyDeviceToHost, s), "D2H offsets")) !=
          TN_OK)
        return st;
      if ((st = cuda_check(cudaStreamSynchronize(s), "offsets sync")) != TN_OK) return st;
      std::vector<size_t> o_t(ns, 0);
      size_t tb = 0;
      for (int c = 0; c < ns; ++c) {
        o_t[c] = tb;
        tb += ((size_t)sp.sec[c].R * (hoff[c + 1] - hoff[c]) * 16 + 255) & ~(size_t)255;
      }
      char* Tb = nullptr;
      if ((st = grow(X.gbuf[2], X.gcap[2], std::max<size_t>(tb, 256), &Tb)) != TN_OK) return st;
      cublasSetStream(X.hb[0], s);
      const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
      BformPtrs bp{};
      for (int c = 0; c < ns; ++c) {
        const int kc = hoff[c + 1] - hoff[c];
        bp.t[c] = reinterpret_cast<const double2*>(Tb + o_t[c]);
        if (kc == 0) continue;
        const SvdSector& S = sp.sec[c];
        const cublasStatus_t b = cublasZgemm(
            X.hb[0], CUBLAS_OP_C, CUBLAS_OP_N, kc, S.R, S.C, &one, reinterpret_cast<const cuDoubleComplex*>(S.ux), S.C,
            reinterpret_cast<const cuDoubleComplex*>(theta[c]), S.C, &zero, reinterpret_cast<cuDoubleComplex*>(Tb + o_t[c]),
            kc);
        if (b != CUBLAS_STATUS_SUCCESS) {
          cublasSetStream(X.hb[0], X.st[0]);
          return fail(TN_ERR_CUDA, "tn_svd_truncate_bform: ZGEMM Θ·V failed in sector " + std::to_string(c));
        }
      }
      cublasSetStream(X.hb[0], X.st[0]);
      k_svd_bform<<<dim3(std::max(1, 2 * p->sm_count / std::max(1, ns) + 1), ns), 256, 0, s>>>(
          sp, bp, d_off, p->d_perm[0], p->d_perm[2], lambda_l, chi_new, p->chi[2],
          reinterpret_cast<double2*>(gamma_k_new), reinterpret_cast<double2*>(gamma_k1_new));
      if ((st = cuda_check(cudaGetLastError(), "SVD factors (B form)")) != TN_OK) return st;
    }
    // k_svd_factors reads the process-wide scratch (X.buf, gbuf): drain it before another call (on any stream
    // or thread) may overwrite that scratch — negligible next to the SVD itself
    if ((st = cuda_check(cudaStreamSynchronize(s), "SVD factors sync")) != TN_OK) return st;
  }
  if ((st = cuda_check(plan_touch(p, s), "plan fence")) != TN_OK) return st;
  *chi_out = res[0];
  std::memcpy(discarded, &res[1], 8);
  return TN_OK;
}

extern "C" tn_status tn_svd_truncate(const tn_plan* p, tn_stream stream, double* const* theta, const double* lambda_l,
                                     const double* lambda_r, int64_t chi_max, double cutoff, int32_t* q_new,
                                     double* lambda_new, double* gamma_k_new, double* gamma_k1_new, int64_t* chi_out,
                                     double* discarded) {
  return svd_truncate_impl(p, stream, theta, lambda_l, lambda_r, chi_max, cutoff, q_new, lambda_new, gamma_k_new,
                           gamma_k1_new, chi_out, discarded, 0);
}

extern "C" tn_status tn_svd_truncate_bform(const tn_plan* p, tn_stream stream, double* const* theta,
                                           const double* lambda_l, int64_t chi_max, double cutoff, int32_t* q_new,
                                           double* lambda_new, double* b_k_new, double* b_k1_new, int64_t* chi_out,
                                           double* discarded) {
  return svd_truncate_impl(p, stream, theta, lambda_l, nullptr, chi_max, cutoff, q_new, lambda_new, b_k_new, b_k1_new,
                           chi_out, discarded, 1);
}
