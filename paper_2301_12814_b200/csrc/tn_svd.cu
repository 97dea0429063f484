// SVD step after Θ: per-sector SVD, global top-χ, new canonical factors.
//
// PAPER.md:67 "Singular value decompositions are then performed on Θ(c^{[k]}), and the largest χ singular
// values out of the singular values for all Θ(c^{[k]}) and their corresponding bonds are retained";
// PAPER.md:192 (SVD "takes up the majority" of GPU time); contract SPEC.md:70-78, tie-break SPEC.md:97.
//
// B200 design (DESIGN.md §4 "SVD step"):
//  * Per-sector SVD with cuSOLVER (polar-decomposition Xgesvdp by default, one-sided Jacobi gesvdj with
//    TN_SVD_ALGO=gesvdj), econ: a library routine, as the paper treats SVD ("a well-researched and
//    optimized routine"). Sectors run concurrently on 8 lanes (handle + stream + host
//    thread each), largest first onto the least-loaded lane. Θ(c) is row-major, i.e. the column-major
//    C×R matrix X = Θᵀ = U_x S V_xᴴ, so Θ = conj(V_x) S U_xᵀ.
//  * Global ranking on the device: one stable radix sort (cub) of all singular values, descending, whose
//    input order is (charge asc, index asc) — exactly SPEC.md:97's tie-break; the kept set is a prefix.
//  * K_sel (one CTA): kept count per charge, discarded weight Σ dropped s², new-bond offsets (charge
//    ascending, then value descending = a prefix of every sector's spectrum), q_new and λ_new.
//  * K_fac: Γ^{[k]}_new[α, a] = U_c[α, s]/λl[α] and Γ^{[k+1]}_new[a, β] = V_c†[s, β]/λr[β] (x/0 := 0),
//    written straight into the caller's bond order through perm_l / perm_r.
#include <cub/device/device_radix_sort.cuh>
#include <cusolverDn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include "tn_internal.cuh"

namespace tn {

namespace {
constexpr int SVD_LANES = 8;  // concurrent sector SVDs (one cuSOLVER handle + stream + host thread each)
struct SvdCtx {  // cuSOLVER handles / streams + a grow-only device scratch, per process and bound to the
                 // device current at first use (one process per GPU, as everywhere in this library)
  cusolverDnHandle_t h[SVD_LANES] = {};
  cudaStream_t st[SVD_LANES] = {};
  cudaEvent_t ev[SVD_LANES + 1] = {};
  gesvdjInfo_t params = nullptr;
  cusolverDnParams_t xparams = nullptr;
  void* buf = nullptr;
  size_t cap = 0;
  std::mutex mu;
};
SvdCtx& ctx() {
  static SvdCtx c;
  return c;
}
// 1: polar-decomposition SVD (Xgesvdp, default: 0.95 s at config 3), 0: one-sided Jacobi (gesvdj, 1.98 s);
// both meet the parity bar (tests/test_gpu_svd.py runs with either)
int svd_algo() {
  static const int v = [] {
    const char* e = getenv("TN_SVD_ALGO");
    return (e && std::string(e) == "gesvdj") ? 0 : 1;
  }();
  return v;
}
}  // namespace

struct SvdSector {          // device views of one sector's SVD
  const double2* ux;        // C × k column-major (ld C)
  const double2* vx;        // R × k column-major (ld R)
  const double* s;          // k values, descending
  int64_t row0, col0;       // sorted positions of Θ(c)'s first row / column
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
      const int32_t al = perm_l[S.row0 + r];
      const double l = lam_l[al];
      const double2 v = S.vx[r + (int64_t)s * S.R];
      const double inv = l != 0.0 ? 1.0 / l : 0.0;
      gk_new[(int64_t)al * ld_k + a0 + s] = make_double2(v.x * inv, -v.y * inv);
    } else {       // V_Θ†[s, col] = U_x[col, s]
      const int64_t j = i - na;
      const int s = (int)(j / S.C), col = (int)(j - (int64_t)s * S.C);
      const int32_t be = perm_r[S.col0 + col];
      const double l = lam_r[be];
      const double2 u = S.ux[col + (int64_t)s * S.C];
      const double inv = l != 0.0 ? 1.0 / l : 0.0;
      gk1_new[(int64_t)(a0 + s) * chi_r + be] = make_double2(u.x * inv, u.y * inv);
    }
  }
}

}  // namespace tn

using namespace tn;

extern "C" tn_status tn_svd_truncate(const tn_plan* p, tn_stream stream, double* const* theta, const double* lambda_l,
                                     const double* lambda_r, int64_t chi_max, double cutoff, int32_t* q_new,
                                     double* lambda_new, double* gamma_k_new, double* gamma_k1_new, int64_t* chi_out,
                                     double* discarded) {
  if (chi_max < 1 || !(cutoff >= 0.0)) return fail(TN_ERR_DOMAIN, "tn_svd_truncate: chi_max < 1 or cutoff < 0");
  if (!p || !theta || !lambda_l || !lambda_r || !q_new || !lambda_new || !gamma_k_new || !gamma_k1_new || !chi_out ||
      !discarded)
    return fail(TN_ERR_DIMENSION, "tn_svd_truncate: NULL argument");
  if (p->world != 1 || p->pair)
    return fail(TN_ERR_UNSUPPORTED, "tn_svd_truncate: needs a single-GPU, single-charge plan (full sectors)");
  cudaStream_t s = (cudaStream_t)stream;
  SvdCtx& X = ctx();
  std::lock_guard<std::mutex> lock(X.mu);
  if (!X.h[0]) {
    for (int i = 0; i < SVD_LANES; ++i) {
      if (cusolverDnCreate(&X.h[i]) != CUSOLVER_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "cusolverDnCreate failed");
      if (cudaStreamCreateWithFlags(&X.st[i], cudaStreamNonBlocking) != cudaSuccess)
        return fail(TN_ERR_CUDA, "SVD stream create failed");
      cusolverDnSetStream(X.h[i], X.st[i]);
    }
    for (auto& e : X.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return fail(TN_ERR_CUDA, "event");
    if (cusolverDnCreateGesvdjInfo(&X.params) != CUSOLVER_STATUS_SUCCESS)
      return fail(TN_ERR_CUDA, "cusolverDnCreateGesvdjInfo failed");
    cusolverDnXgesvdjSetTolerance(X.params, 0.0);      // 0 → machine accuracy
    cusolverDnXgesvdjSetMaxSweeps(X.params, 100);
    if (cusolverDnCreateParams(&X.xparams) != CUSOLVER_STATUS_SUCCESS) return fail(TN_ERR_CUDA, "cusolver params");
  }
  const int algo = svd_algo();
  const int ns = p->nsec;
  // ---- scratch layout: per sector U_x, V_x, S, workspace; then sort buffers ----
  SvdParams sp{};
  sp.nsec = ns;
  std::vector<size_t> o_ux(ns), o_vx(ns), o_s(ns), o_w(ns);
  std::vector<int> lwork(ns, 0);
  std::vector<size_t> hbytes(ns, 0), wsz(ns, 0);
  std::vector<int64_t> base(ns + 1, 0);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  for (int c = 0; c < ns; ++c) {
    const int R = (int)p->R[c], C = (int)p->C[c], k = std::min(R, C);
    base[c + 1] = base[c] + k;
    if (k == 0) continue;
    size_t wbytes = 0;
    if (algo == 0) {
      if (cusolverDnZgesvdj_bufferSize(X.h[0], CUSOLVER_EIG_MODE_VECTOR, 1, C, R, nullptr, C, nullptr, nullptr, C,
                                       nullptr, R, &lwork[c], X.params) != CUSOLVER_STATUS_SUCCESS)
        return fail(TN_ERR_CUDA, "cusolverDnZgesvdj_bufferSize failed");
      wbytes = (size_t)lwork[c] * 16;
    } else {
      size_t hb = 0;
      if (cusolverDnXgesvdp_bufferSize(X.h[0], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, C, R, CUDA_C_64F, nullptr, C,
                                       CUDA_R_64F, nullptr, CUDA_C_64F, nullptr, C, CUDA_C_64F, nullptr, R, CUDA_C_64F,
                                       &wbytes, &hb) != CUSOLVER_STATUS_SUCCESS)
        return fail(TN_ERR_CUDA, "cusolverDnXgesvdp_bufferSize failed");
      hbytes[c] = hb;
    }
    o_ux[c] = take((size_t)C * k * 16);
    o_vx[c] = take((size_t)R * k * 16);
    o_s[c] = take((size_t)k * 8);
    o_w[c] = take(wbytes);
    wsz[c] = wbytes;
  }
  const int64_t total_max = base[ns];
  const size_t o_info = take((size_t)ns * 4);
  const size_t o_n2 = take((size_t)ns * 8);
  const size_t o_kin = take((size_t)std::max<int64_t>(total_max, 1) * 8),
               o_kout = take((size_t)std::max<int64_t>(total_max, 1) * 8);
  const size_t o_vin = take((size_t)std::max<int64_t>(total_max, 1) * 4),
               o_vout = take((size_t)std::max<int64_t>(total_max, 1) * 4);
  const size_t o_base = take((size_t)(ns + 1) * 8);
  const size_t o_off = take((size_t)(ns + 1) * 4);
  const size_t o_res = take(16);
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const double*)nullptr, (double*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(total_max, 1));
  const size_t o_sort = take(sort_bytes);
  if (off > X.cap) {
    if (X.buf) cudaFree(X.buf);
    X.buf = nullptr;
    X.cap = 0;
    if (cudaMalloc(&X.buf, off) != cudaSuccess) return fail(TN_ERR_OOM, "tn_svd_truncate: scratch allocation");
    X.cap = off;
  }
  char* B = static_cast<char*>(X.buf);
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
    if (k == 0) continue;
    if (!theta[c]) return fail(TN_ERR_DIMENSION, "tn_svd_truncate: NULL Θ(c) for a non-empty sector");
    S.ux = reinterpret_cast<double2*>(B + o_ux[c]);
    S.vx = reinterpret_cast<double2*>(B + o_vx[c]);
    S.s = reinterpret_cast<double*>(B + o_s[c]);
    order.push_back(c);
  }
  tn_status st = cuda_check(cudaMemsetAsync(d_info, 0, ns * sizeof(int), s), "memset info");  // empty sectors
  if (st != TN_OK) return st;
  std::vector<std::string> errs(SVD_LANES);
  // one wave of sector SVDs: largest first, greedy onto the least-loaded lane (cost ~ R·C·min(R, C))
  auto run_wave = [&](std::vector<int> wave) -> tn_status {
    if (wave.empty()) return TN_OK;
    std::sort(wave.begin(), wave.end(), [&](int a, int b) {
      return (double)p->R[a] * p->C[a] * std::min(p->R[a], p->C[a]) >
             (double)p->R[b] * p->C[b] * std::min(p->R[b], p->C[b]);
    });
    std::vector<std::vector<int>> lane(SVD_LANES);
    double load[SVD_LANES] = {};
    for (int c : wave) {
      const int l = (int)(std::min_element(load, load + SVD_LANES) - load);
      lane[l].push_back(c);
      load[l] += (double)p->R[c] * p->C[c] * std::min(p->R[c], p->C[c]);
    }
    tn_status r0 = cuda_check(cudaEventRecord(X.ev[SVD_LANES], s), "Θ ready");
    if (r0 != TN_OK) return r0;
    auto work = [&](int l) {
      if (cudaStreamWaitEvent(X.st[l], X.ev[SVD_LANES], 0) != cudaSuccess) {
        errs[l] = "stream wait";
        return;
      }
      std::vector<char> hbuf;
      for (int c : lane[l]) {
        const SvdSector& S = sp.sec[c];
        const int R = S.R, C = S.C;
        cusolverStatus_t r;
        // X = Θᵀ (column-major C × R, ld C) = U_x S V_xᴴ; Θ(c) is destroyed
        if (algo == 0) {
          r = cusolverDnZgesvdj(X.h[l], CUSOLVER_EIG_MODE_VECTOR, 1, C, R, reinterpret_cast<cuDoubleComplex*>(theta[c]),
                                C, const_cast<double*>(S.s),
                                reinterpret_cast<cuDoubleComplex*>(const_cast<double2*>(S.ux)), C,
                                reinterpret_cast<cuDoubleComplex*>(const_cast<double2*>(S.vx)), R,
                                reinterpret_cast<cuDoubleComplex*>(B + o_w[c]), lwork[c], d_info + c, X.params);
        } else {
          hbuf.resize(std::max<size_t>(hbytes[c], 1));
          double herr = 0.0;
          r = cusolverDnXgesvdp(X.h[l], X.xparams, CUSOLVER_EIG_MODE_VECTOR, 1, C, R, CUDA_C_64F, theta[c], C,
                                CUDA_R_64F, const_cast<double*>(S.s), CUDA_C_64F, const_cast<double2*>(S.ux), C,
                                CUDA_C_64F, const_cast<double2*>(S.vx), R, CUDA_C_64F, B + o_w[c], wsz[c], hbuf.data(),
                                hbytes[c], d_info + c, &herr);
        }
        if (r != CUSOLVER_STATUS_SUCCESS) {
          errs[l] = "cuSOLVER SVD failed in sector " + std::to_string(c) + " (status " + std::to_string((int)r) + ")";
          return;
        }
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
      if ((r0 = cuda_check(cudaStreamWaitEvent(s, X.ev[l], 0), "join SVD lanes")) != TN_OK) return r0;
    }
    return TN_OK;
  };
  // ---- norm bound: SVD the heaviest sectors first; a sector with ‖Θ(c)‖_F below the χ-th largest singular
  // value found so far cannot place any value in the global top χ (that threshold only grows), so its SVD
  // is skipped and its whole weight ‖Θ(c)‖²_F is discarded — the result is identical ----
  double disc_skipped = 0.0;
  {
    ThetaPtrs tp{};
    for (int c = 0; c < ns; ++c) {
      tp.p[c] = reinterpret_cast<const double2*>(theta[c]);
      tp.n[c] = sp.sec[c].k ? (int64_t)p->R[c] * p->C[c] : 0;
    }
    double* d_n2 = reinterpret_cast<double*>(B + o_n2);
    if ((st = cuda_check(cudaMemsetAsync(d_n2, 0, ns * sizeof(double), s), "memset norms")) != TN_OK) return st;
    k_sector_norm2<<<dim3(32, ns), 256, 0, s>>>(tp, d_n2);
    std::vector<double> n2(ns);
    if ((st = cuda_check(cudaMemcpyAsync(n2.data(), d_n2, ns * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H norms")) !=
        TN_OK)
      return st;
    if ((st = cuda_check(cudaStreamSynchronize(s), "norm sync")) != TN_OK) return st;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return n2[a] > n2[b]; });
    std::vector<int> wave1, rest;
    int64_t have = 0;
    for (int c : order) {
      if (have < 2 * chi_max) {
        wave1.push_back(c);
        have += sp.sec[c].k;
      } else {
        rest.push_back(c);
      }
    }
    if ((st = run_wave(wave1)) != TN_OK) return st;
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
      if ((st = run_wave(wave2)) != TN_OK) return st;
    }
    for (int c = 0; c < ns; ++c) base[c + 1] = base[c] + sp.sec[c].k;
  }
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
    k_svd_factors<<<dim3(std::max(1, 2 * p->sm_count / std::max(1, ns) + 1), ns), 256, 0, s>>>(
        sp, d_off, p->d_perm[0], p->d_perm[2], lambda_l, lambda_r, chi_new, p->chi[2],
        reinterpret_cast<double2*>(gamma_k_new), reinterpret_cast<double2*>(gamma_k1_new));
    if ((st = cuda_check(cudaGetLastError(), "SVD factors")) != TN_OK) return st;
  }
  *chi_out = res[0];
  std::memcpy(discarded, &res[1], 8);
  return TN_OK;
}
