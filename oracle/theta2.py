"""Plain CPU oracle of the MPO (doubled-charge) Θ(c1, c2) — TEST INFRASTRUCTURE ONLY (see __init__).

PAPER.md:107 (Supp. §1.6, "Adaptation to MPO Gaussian boson sampling"): "MPOs are vectorized into the
MPS form, U → U⊗U*, and two conserved charges are present. The CPU implementation of the algorithm
now requires loops over two sets of conserved charges". PAPER.md:101: "the overall Θ matrix is
broken up into Θ(c_1^k, c_2^k)'s". SPEC.md:142-150 (double_gate: (U⊗U*)[(a,b),(c,e)] = U[a,c]·
conj(U[b,e])) and SPEC.md:348-356 (apply_gate_mpo: Θ slices indexed by the centre charge pair).

A vectorized site index is the pair (i, i') (ket and bra occupations, each in [0, d−1]); a bond α
carries two charges (c1, c2) = photons to the right in the ket and in the bra copy. Eq. S5 with
U → U⊗U* and one δ pair per species reads

  Θ(c1,c2)[α,β] = λl[α] λr[β] Σ_{α_k} Σ_{j,j'} U^{i_k,i_{k+1}}_{j_k,j_{k+1}} conj(U^{i'_k,i'_{k+1}}_{j'_k,j'_{k+1}})
                  Γk[α,α_k] λk[α_k] Γk1[α_k,β]
                  × δ(l1−m1−j_k) δ(m1−r1−j_{k+1}) δ(l1−c1−i_k) δ(c1−r1−i_{k+1})
                  × δ(l2−m2−j'_k) δ(m2−r2−j'_{k+1}) δ(l2−c2−i'_k) δ(c2−r2−i'_{k+1}),

(l, m, r) = the charge pairs of (α, α_k, β). Readings (R16–R18): bonds are sorted
lexicographically by (c1, c2), stable ("Pair-charge ordering … lexicographic (c1 major,
c2 minor)"); Θ(c1,c2) is compact row-major, rows = sorted left positions with both l1−c1 and l2−c2 in
[0, d−1] (in sorted order), columns likewise with c1−r1, c2−r2 ∈ [0, d−1].
The loop below is the literal six-charge loop ("loops over two sets of conserved charges").
"""
from __future__ import annotations

import numpy as np

from .theta import bs_unitary_block


def sort_pair_bonds(q1, q2):
    """Stable lexicographic sort of one bond by its charge pair (c1 major, c2 minor).
    Returns perm (sorted position → original index) as int32."""
    q1 = [int(x) for x in q1]
    q2 = [int(x) for x in q2]
    return np.array(sorted(range(len(q1)), key=lambda i: (q1[i], q2[i])), dtype=np.int32)


def pair_sector_rows(q1s, q2s, d, c1, c2):
    """Sorted positions (ascending) of the left bonds admissible for Θ(c1,c2): l − c ∈ [0, d−1]²."""
    return np.array([p for p in range(len(q1s)) if 0 <= q1s[p] - c1 <= d - 1 and 0 <= q2s[p] - c2 <= d - 1],
                    dtype=np.int64)


def pair_sector_cols(q1s, q2s, d, c1, c2):
    """Sorted positions of the right bonds admissible for Θ(c1,c2): c − r ∈ [0, d−1]²."""
    return np.array([p for p in range(len(q1s)) if 0 <= c1 - q1s[p] <= d - 1 and 0 <= c2 - q2s[p] <= d - 1],
                    dtype=np.int64)


def theta2_sectors(N, d, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r, gamma_k, lam_k, gamma_k1, lam_l, lam_r, theta, phi,
                   u_blocks=None, sectors=None):
    """Θ(c1, c2) for every (c1, c2) ∈ [0, N]², by the literal loop over the three charge pairs.

    Returns (secs, perms, u_blocks): secs[(c1, c2)] = complex128[R, C] in sorted bond order (None when
    not requested via `sectors`), perms = (perm_l, perm_c, perm_r)."""
    perm_l = sort_pair_bonds(q1_l, q2_l)
    perm_c = sort_pair_bonds(q1_c, q2_c)
    perm_r = sort_pair_bonds(q1_r, q2_r)
    l1, l2 = np.asarray(q1_l)[perm_l], np.asarray(q2_l)[perm_l]
    m1, m2 = np.asarray(q1_c)[perm_c], np.asarray(q2_c)[perm_c]
    r1, r2 = np.asarray(q1_r)[perm_r], np.asarray(q2_r)[perm_r]
    Gk = np.asarray(gamma_k)[perm_l][:, perm_c]
    Gk1 = np.asarray(gamma_k1)[perm_c][:, perm_r]
    lk = np.asarray(lam_k)[perm_c]
    ll = np.asarray(lam_l)[perm_l]
    lr = np.asarray(lam_r)[perm_r]
    if u_blocks is None:
        u_blocks = [bs_unitary_block(n, theta, phi, d) for n in range(min(N, 2 * d - 2) + 1)]

    def U(n, i, j):                      # ⟨i, n−i|U|j, n−j⟩
        lo = max(0, n - d + 1)
        return u_blocks[n][i - lo, j - lo]

    def seg(a1, a2, x1, x2):             # sorted positions of one charge pair (contiguous after sorting)
        idx = np.nonzero((a1 == x1) & (a2 == x2))[0]
        return idx

    wanted = None if sectors is None else set(tuple(s) for s in sectors)
    rng = range(N + 1)
    out = {}
    for c1 in rng:
        for c2 in rng:
            if wanted is not None and (c1, c2) not in wanted:
                out[(c1, c2)] = None
                continue
            rows = pair_sector_rows(l1, l2, d, c1, c2)
            cols = pair_sector_cols(r1, r2, d, c1, c2)
            th = np.zeros((len(rows), len(cols)), dtype=np.complex128)
            rloc = {p: i for i, p in enumerate(rows)}
            cloc = {p: i for i, p in enumerate(cols)}
            for cl1 in range(c1, min(N, c1 + d - 1) + 1):              # i_k  = l1 − c1
                for cl2 in range(c2, min(N, c2 + d - 1) + 1):          # i'_k = l2 − c2
                    sl = seg(l1, l2, cl1, cl2)
                    if len(sl) == 0:
                        continue
                    for cr1 in range(max(0, c1 - d + 1), c1 + 1):      # i_{k+1}  = c1 − r1
                        for cr2 in range(max(0, c2 - d + 1), c2 + 1):  # i'_{k+1} = c2 − r2
                            sr = seg(r1, r2, cr1, cr2)
                            if len(sr) == 0:
                                continue
                            for cc1 in range(cr1, cl1 + 1):
                                if cl1 - cc1 > d - 1 or cc1 - cr1 > d - 1:  # j_k, j_{k+1} ∈ [0, d−1]
                                    continue
                                for cc2 in range(cr2, cl2 + 1):
                                    if cl2 - cc2 > d - 1 or cc2 - cr2 > d - 1:
                                        continue
                                    sc = seg(m1, m2, cc1, cc2)
                                    if len(sc) == 0:
                                        continue
                                    w = U(cl1 - cr1, cl1 - c1, cl1 - cc1) * np.conj(U(cl2 - cr2, cl2 - c2, cl2 - cc2))
                                    blk = (Gk[np.ix_(sl, sc)] * lk[sc][None, :]) @ Gk1[np.ix_(sc, sr)]
                                    ri = [rloc[p] for p in sl]
                                    ci = [cloc[p] for p in sr]
                                    th[np.ix_(ri, ci)] += w * blk
            th *= ll[rows][:, None] * lr[cols][None, :]
            out[(c1, c2)] = th
    return out, (perm_l, perm_c, perm_r), u_blocks


def flop_counts2(N, d, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r):
    """Useful work of the pair path, 8 real flops per complex MAC:
    F_contract = 8 Σ_{allowed (l, m, r)} n_l n_m n_r over charge PAIRS (the §8(d) definition);
    F_mix = 8 Σ_{(l, r)} n_l n_r (L1²L2 + L1L2²), L_s = #valid c_s of species s — the U⊗U* mix applied
    one species at a time (U_{n1} along c1, then conj(U_{n2}) along c2; DESIGN.md §4 "K5P")."""
    def counts(a, b):
        h = {}
        for x, y in zip(np.asarray(a).tolist(), np.asarray(b).tolist()):
            h[(x, y)] = h.get((x, y), 0) + 1
        return h
    nl, nm, nr = counts(q1_l, q2_l), counts(q1_c, q2_c), counts(q1_r, q2_r)
    ok = lambda a, b: 0 <= a - b <= d - 1
    fc = fm = 0
    for (a1, a2), nla in nl.items():
        for (b1, b2), nrb in nr.items():
            L1 = sum(1 for x in range(N + 1) if ok(a1, x) and ok(x, b1))
            L2 = sum(1 for y in range(N + 1) if ok(a2, y) and ok(y, b2))
            for (x, y), nmm in nm.items():
                if ok(a1, x) and ok(x, b1) and ok(a2, y) and ok(y, b2):
                    fc += 8 * nla * nmm * nrb
            if L1 and L2:
                fm += 8 * nla * nrb * (L1 * L1 * L2 + L1 * L2 * L2)
    return int(fc), int(fm)


def theta2_element(N, d, c1, c2, a, b, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r, gamma_k, lam_k, gamma_k1, lam_l, lam_r,
                   u_blocks, perms):
    """One element Θ(c1,c2)[a, b] (local indices in sorted order) by the same literal sum — sampled parity at
    sizes where the full loop is too slow. `perms` = (perm_l, perm_c, perm_r) from sort_pair_bonds."""
    perm_l, perm_c, perm_r = perms
    l1s, l2s = np.asarray(q1_l)[perm_l], np.asarray(q2_l)[perm_l]
    r1s, r2s = np.asarray(q1_r)[perm_r], np.asarray(q2_r)[perm_r]
    al = int(perm_l[pair_sector_rows(l1s, l2s, d, c1, c2)[a]])
    be = int(perm_r[pair_sector_cols(r1s, r2s, d, c1, c2)[b]])
    l1, l2, r1, r2 = int(q1_l[al]), int(q2_l[al]), int(q1_r[be]), int(q2_r[be])

    def U(n, i, j):
        lo = max(0, n - d + 1)
        return u_blocks[n][i - lo, j - lo]

    m1s, m2s = np.asarray(q1_c), np.asarray(q2_c)
    acc = 0j
    for cc1 in range(r1, l1 + 1):
        if l1 - cc1 > d - 1 or cc1 - r1 > d - 1:
            continue
        for cc2 in range(r2, l2 + 1):
            if l2 - cc2 > d - 1 or cc2 - r2 > d - 1:
                continue
            g = np.nonzero((m1s == cc1) & (m2s == cc2))[0]
            if len(g) == 0:
                continue
            w = U(l1 - r1, l1 - c1, l1 - cc1) * np.conj(U(l2 - r2, l2 - c2, l2 - cc2))
            acc += w * np.sum(gamma_k[al, g] * lam_k[g] * gamma_k1[g, be])
    return acc * lam_l[al] * lam_r[be]
