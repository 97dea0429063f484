"""Plain CPU oracle of the charge-sectored two-site Θ(c) (TEST INFRASTRUCTURE ONLY; see __init__).

Notation follows PAPER.md Supplementary §1.1:
  c_l = c^{[k-1]}_{α_{k-1}}, c_c = c^{[k]}_{α_k}, c_r = c^{[k+1]}_{α_{k+1}}  (photons to the right)
  Eq. S5:
    Θ(c)[α,β] = Σ_{j_k,j_{k+1}} Σ_{α_k} U^{i_k,i_{k+1}}_{j_k,j_{k+1}} λl[α] Γk[α,α_k] λk[α_k] Γk1[α_k,β] λr[β]
                × δ(c_l − c_c − j_k) δ(c_c − c_r − j_{k+1}) δ(c_l − c − i_k) δ(c − c_r − i_{k+1})
  with 0 ≤ c ≤ N and 0 ≤ i, j ≤ d−1.
"""
from __future__ import annotations

import math

import mpmath
import numpy as np


# ----------------------------------------------------------------------------------------------
# Bond sorting
# ----------------------------------------------------------------------------------------------
def sort_bonds(q, N: int):
    """Stable ascending sort of one bond by charge.

    Returns (perm, off): perm[p] = original bond index at sorted position p (Python's `sorted` is
    stable); off[q] = number of bonds with charge < q for q = 0..N+1 (length N+2).
    """
    q = [int(x) for x in q]
    perm = sorted(range(len(q)), key=q.__getitem__)
    off = [0] * (N + 2)
    for qq in range(N + 2):
        off[qq] = sum(1 for x in q if x < qq)
    return np.array(perm, dtype=np.int32), np.array(off, dtype=np.int32)


# ----------------------------------------------------------------------------------------------
# Beam-splitter unitary in the Fock basis (Eq. S4; convention DESIGN.md R5)
# ----------------------------------------------------------------------------------------------
def _u_element_mp(n: int, i: int, j: int, theta: float, phi: float):
    """⟨i, n−i| exp[θ(e^{iφ} a†b − e^{−iφ} a b†)] |j, n−j⟩ at the current mpmath precision.

    Derivation (R5): B a† B† = cosθ a† − e^{−iφ} sinθ b†, B b† B† = cosθ b† + e^{iφ} sinθ a†;
    expanding B (a†)^j (b†)^{n−j}|0⟩ / √(j!(n−j)!) binomially gives
      U_n[i][j] = e^{iφ(i−j)} √(i!(n−i)!/(j!(n−j)!)) Σ_k C(j,k) C(n−j,i−k) (−1)^{j−k} cos^{n−j−i+2k}θ sin^{i+j−2k}θ.
    """
    th = mpmath.mpf(theta)
    ph = mpmath.mpf(phi)
    c, s = mpmath.cos(th), mpmath.sin(th)
    acc = mpmath.mpf(0)
    for k in range(0, j + 1):
        l = i - k
        if l < 0 or l > n - j:
            continue
        term = mpmath.binomial(j, k) * mpmath.binomial(n - j, l)
        term *= c ** (n - j - i + 2 * k) * s ** (i + j - 2 * k)
        if (j - k) % 2:
            term = -term
        acc += term
    pref = mpmath.sqrt(mpmath.factorial(i) * mpmath.factorial(n - i)
                       / (mpmath.factorial(j) * mpmath.factorial(n - j)))
    return mpmath.exp(1j * ph * (i - j)) * pref * acc


def bs_unitary_block(n: int, theta: float, phi: float, d: int, dps: int = 50) -> np.ndarray:
    """Block U_n of fixed total photon number n, restricted to occupations ≤ d−1 (R6).

    Rows/cols are i = i_k (resp. j = j_k) in [lo_n, hi_n], lo_n = max(0, n−d+1), hi_n = min(n, d−1);
    entry [i−lo_n][j−lo_n] = ⟨i, n−i|U|j, n−j⟩. Evaluated at `dps` digits, rounded once to complex128.
    """
    lo, hi = max(0, n - d + 1), min(n, d - 1)
    s = hi - lo + 1
    out = np.zeros((s, s), dtype=np.complex128)
    with mpmath.workdps(dps):
        for i in range(lo, hi + 1):
            for j in range(lo, hi + 1):
                v = _u_element_mp(n, i, j, theta, phi)
                out[i - lo, j - lo] = complex(float(mpmath.re(v)), float(mpmath.im(v)))
    return out


def packed_u_offsets(d: int, N: int):
    """Block start offsets of the packed U (SURVEY.md §8(c) 'Packed U'); returns (starts, total)."""
    n_max = min(N, 2 * d - 2)
    starts, tot = [], 0
    for n in range(n_max + 1):
        s = min(n, d - 1) - max(0, n - d + 1) + 1
        starts.append(tot)
        tot += s * s
    return starts, tot


def packed_u(theta: float, phi: float, d: int, N: int, dps: int = 50) -> np.ndarray:
    """All blocks n = 0..min(N, 2d−2) concatenated, each row-major [i][j]."""
    n_max = min(N, 2 * d - 2)
    return np.concatenate([bs_unitary_block(n, theta, phi, d, dps).ravel() for n in range(n_max + 1)])


# ----------------------------------------------------------------------------------------------
# Θ(c) by the literal triple charge loop
# ----------------------------------------------------------------------------------------------
def sector_ranges(off_l, off_r, N: int, d: int, c: int):
    """Sorted-position row range and column range of Θ(c) (R2):
    rows: c ≤ c_l ≤ c+d−1 (i_k = c_l − c ∈ [0,d−1]); cols: c−d+1 ≤ c_r ≤ c (i_{k+1} = c − c_r ∈ [0,d−1])."""
    r0, r1 = int(off_l[c]), int(off_l[min(N, c + d - 1) + 1])
    k0, k1 = int(off_r[max(0, c - d + 1)]), int(off_r[c + 1])
    return (r0, r1), (k0, k1)


def _u_lookup(blocks, d, n, i, j):
    lo = max(0, n - d + 1)
    return blocks[n][i - lo, j - lo]


def theta_sectors(N, d, q_l, q_c, q_r, gamma_k, lam_k, gamma_k1, lam_l, lam_r, theta, phi,
                  u_blocks=None, sectors=None):
    """Θ(c) for c = 0..N, literally as PAPER.md:72 describes.

    'looping through all possible left, center and right charges c_l, c_c, c_r … choose the correct
    entry of U, which takes care of the sum over the j indices, and the rest of the contraction is
    only over α_k.' Rows/cols of Θ(c) are in sorted bond order (R2); returns
    (sectors, perms, offs, u_blocks) with sectors[c] a complex128[R_c, C_c] array. If `sectors` (an
    iterable of c) is given only those are computed (others are None) — a bounded sample for timing.
    """
    perm_l, off_l = sort_bonds(q_l, N)
    perm_c, off_c = sort_bonds(q_c, N)
    perm_r, off_r = sort_bonds(q_r, N)
    Gk = np.asarray(gamma_k)[perm_l][:, perm_c]
    Gk1 = np.asarray(gamma_k1)[perm_c][:, perm_r]
    lk = np.asarray(lam_k)[perm_c]
    ll = np.asarray(lam_l)[perm_l]
    lr = np.asarray(lam_r)[perm_r]
    if u_blocks is None:
        u_blocks = [bs_unitary_block(n, theta, phi, d) for n in range(min(N, 2 * d - 2) + 1)]

    def seg(off, q):
        return slice(int(off[q]), int(off[q + 1]))

    wanted = set(range(N + 1)) if sectors is None else set(int(c) for c in sectors)
    sectors = []
    for c in range(N + 1):
        if c not in wanted:
            sectors.append(None)
            continue
        (r0, r1), (k0, k1) = sector_ranges(off_l, off_r, N, d, c)
        th = np.zeros((r1 - r0, k1 - k0), dtype=np.complex128)
        for c_l in range(c, min(N, c + d - 1) + 1):              # i_k = c_l − c
            for c_r in range(max(0, c - d + 1), c + 1):          # i_{k+1} = c − c_r
                n = c_l - c_r
                for c_c in range(c_r, c_l + 1):
                    if c_l - c_c > d - 1 or c_c - c_r > d - 1:   # j_k, j_{k+1} ∈ [0, d−1]
                        continue
                    w = _u_lookup(u_blocks, d, n, c_l - c, c_l - c_c)
                    sl, sc, sr = seg(off_l, c_l), seg(off_c, c_c), seg(off_r, c_r)
                    blk = (Gk[sl, sc] * lk[sc][None, :]) @ Gk1[sc, sr]
                    th[sl.start - r0:sl.stop - r0, sr.start - k0:sr.stop - k0] += w * blk
        th *= ll[r0:r1][:, None] * lr[k0:k1][None, :]
        sectors.append(th)
    return sectors, (perm_l, perm_c, perm_r), (off_l, off_c, off_r), u_blocks


def theta_element(N, d, c, a, b, q_l, q_c, q_r, gamma_k, lam_k, gamma_k1, lam_l, lam_r, u_blocks,
                  sorted_tables):
    """One element Θ(c)[a, b] (local indices) by the same literal sum, for sampled parity at full size.

    `sorted_tables` = (perms, offs) from `sort_bonds` of each bond.
    """
    (perm_l, perm_c, perm_r), (off_l, off_c, off_r) = sorted_tables
    (r0, _), (k0, _) = sector_ranges(off_l, off_r, N, d, c)
    pa, pb = r0 + a, k0 + b
    al, be = int(perm_l[pa]), int(perm_r[pb])
    c_l, c_r = int(q_l[al]), int(q_r[be])
    n = c_l - c_r
    acc = 0j
    for c_c in range(c_r, c_l + 1):
        if c_l - c_c > d - 1 or c_c - c_r > d - 1:
            continue
        w = _u_lookup(u_blocks, d, n, c_l - c, c_l - c_c)
        g = perm_c[int(off_c[c_c]):int(off_c[c_c + 1])]
        acc += w * np.sum(gamma_k[al, g] * lam_k[g] * gamma_k1[g, be])
    return acc * lam_l[al] * lam_r[be]


# ----------------------------------------------------------------------------------------------
# Useful work; integer-exact, 8 real flops per complex MAC
# ----------------------------------------------------------------------------------------------
def flop_counts(N, d, q_l, q_c, q_r):
    """(F_contract, F_mix, sum_c R_c*C_c) from the per-charge bond counts."""
    nl = np.bincount(np.asarray(q_l), minlength=N + 1).astype(object)
    nc = np.bincount(np.asarray(q_c), minlength=N + 1).astype(object)
    nr = np.bincount(np.asarray(q_r), minlength=N + 1).astype(object)
    f_con, f_mix = 0, 0
    for c_l in range(N + 1):
        for c_r in range(N + 1):
            n = c_l - c_r
            if n < 0 or n > 2 * d - 2:
                continue
            n_valid_c, n_valid_cc = 0, 0
            for c in range(N + 1):
                if 0 <= c_l - c <= d - 1 and 0 <= c - c_r <= d - 1:
                    n_valid_c += 1
                    if nc[c] > 0:
                        n_valid_cc += 1
                        f_con += 8 * nl[c_l] * nc[c] * nr[c_r]
            f_mix += 8 * nl[c_l] * nr[c_r] * n_valid_c * n_valid_cc
    tot = 0
    perm_off_l = np.concatenate([[0], np.cumsum(nl)])
    perm_off_r = np.concatenate([[0], np.cumsum(nr)])
    for c in range(N + 1):
        R = perm_off_l[min(N, c + d - 1) + 1] - perm_off_l[c]
        C = perm_off_r[c + 1] - perm_off_r[max(0, c - d + 1)]
        tot += R * C
    return int(f_con), int(f_mix), int(tot)
