// K2 — Fock-basis beam-splitter U builder (Eq. S4; "O(d^4) for initializing U",
// PAPER.md:70). Only the photon-conserving blocks i_k+i_{k+1} = j_k+j_{k+1} = n are stored (packed
// layout in include/tn_theta.h).
//
// Convention (R5): B = exp[θ(e^{iφ} a†b − e^{−iφ} a b†)], a = mode k. Closed form:
//   U_n[i][j] = e^{iφ(i−j)} √(C(n,j)/C(n,i)) Σ_k (−1)^{j−k} C(j,k) C(n−j,i−k) cos^{n−j−i+2k}θ sin^{i+j−2k}θ
// The alternating sum cancels heavily at large n (terms up to ~3e5 at n = 47, R7), so it
// is evaluated in double-double; binomials are exact unsigned 128-bit integers; cos θ, sin θ and the
// phase are double-accurate (the error they induce is ≤ ~n·1e-16, the closed form being homogeneous
// of degree n in (cos θ, sin θ)). One CTA per block n; latency-bound (≤ 0.6 MB output).
#include "tn_internal.cuh"

namespace tn {

__device__ __forceinline__ dd binom_dd(int n, int k) {
  if (k < 0 || k > n) return {0.0, 0.0};
  if (k > n - k) k = n - k;
  unsigned __int128 c = 1;
  for (int t = 1; t <= k; ++t) c = c * (unsigned __int128)(n - k + t) / (unsigned __int128)t;  // exact
  double hi = (double)c;
  unsigned __int128 hi_i = (unsigned __int128)hi;
  double lo = (c >= hi_i) ? (double)(c - hi_i) : -(double)(hi_i - c);
  return quick_two_sum(hi, lo);
}

__global__ void __launch_bounds__(256) k2_bs_unitary(int d, double theta, double phi,
                                                     double2* __restrict__ U) {
  const int n = blockIdx.x;
  __shared__ dd cpow[2 * TN_MAX_N + 2];
  __shared__ dd spow[2 * TN_MAX_N + 2];
  double s, c;
  sincos(theta, &s, &c);
  if (threadIdx.x == 0) {
    dd cp = dd_from(1.0), sp = dd_from(1.0);
    for (int e = 0; e <= n; ++e) {
      cpow[e] = cp;
      spow[e] = sp;
      cp = dd_mul(cp, dd_from(c));
      sp = dd_mul(sp, dd_from(s));
    }
  }
  __syncthreads();
  const int lo = max(0, n - d + 1), hi = min(n, d - 1);
  const int sn = hi - lo + 1;
  // block start: Σ_{m<n} s_m², recomputed here (n ≤ 2·TN_MAX_N).
  int64_t start = 0;
  for (int m = 0; m < n; ++m) {
    int sm = min(m, d - 1) - max(0, m - d + 1) + 1;
    start += (int64_t)sm * sm;
  }
  for (int e = threadIdx.x; e < sn * sn; e += blockDim.x) {
    const int i = lo + e / sn, j = lo + e % sn;
    dd acc = dd_from(0.0);
    for (int k = 0; k <= j; ++k) {
      const int l = i - k;
      if (l < 0 || l > n - j) continue;
      dd t = dd_mul(binom_dd(j, k), binom_dd(n - j, l));
      t = dd_mul(t, cpow[n - j - i + 2 * k]);
      t = dd_mul(t, spow[i + j - 2 * k]);
      acc = ((j - k) & 1) ? dd_add(acc, dd_neg(t)) : dd_add(acc, t);
    }
    const dd pref = dd_sqrt(dd_div(binom_dd(n, j), binom_dd(n, i)));
    const dd v = dd_mul(pref, acc);
    const double mag = v.hi + v.lo;
    // e^{iφ(i−j)}: argument formed exactly in double-double, then one correction step.
    const dd arg = two_prod(phi, (double)(i - j));
    double sa, ca;
    sincos(arg.hi, &sa, &ca);
    const double cr = ca - arg.lo * sa, si = sa + arg.lo * ca;
    U[start + e] = make_double2(mag * cr, mag * si);
  }
}

cudaError_t launch_bs_unitary(int d, int N, double theta, double phi, const int32_t* ustart_host, double2* U,
                              cudaStream_t s) {
  (void)ustart_host;
  const int nmax = min(N, 2 * d - 2);
  k2_bs_unitary<<<nmax + 1, 256, 0, s>>>(d, theta, phi, U);
  return cudaGetLastError();
}

}  // namespace tn
