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

// binom: (nmax+1)×(nmax+1) table of C(n,k) as double-double pairs (exact below 2^106), built by the
// plan from exact 128-bit integers (host), row-major.
__global__ void __launch_bounds__(256) k2_bs_unitary(int d, int nmax, double theta, double phi,
                                                     const double2* __restrict__ binom, double2* __restrict__ U) {
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
    const int ld = nmax + 1;
    auto B = [&](int nn, int kk) {
      const double2 v = binom[nn * ld + kk];
      return dd{v.x, v.y};
    };
    for (int k = max(0, i - (n - j)); k <= min(j, i); ++k) {
      const int l = i - k;
      dd t = dd_mul(B(j, k), B(n - j, l));
      t = dd_mul(t, cpow[n - j - i + 2 * k]);
      t = dd_mul(t, spow[i + j - 2 * k]);
      acc = ((j - k) & 1) ? dd_add(acc, dd_neg(t)) : dd_add(acc, t);
    }
    const dd pref = dd_sqrt(dd_div(B(n, j), B(n, i)));
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

cudaError_t launch_bs_unitary(int d, int N, double theta, double phi, const double2* binom, double2* U,
                              cudaStream_t s) {
  const int nmax = min(N, 2 * d - 2);
  k2_bs_unitary<<<nmax + 1, 256, 0, s>>>(d, nmax, theta, phi, binom, U);
  return cudaGetLastError();
}

}  // namespace tn
