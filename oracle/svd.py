"""Plain CPU oracle of the per-sector SVD + global top-χ truncation + new bond (TEST INFRASTRUCTURE ONLY).

PAPER.md:67: "Singular value decompositions are then performed on Θ(c^{[k]}), and the largest χ singular
values out of the singular values for all Θ(c^{[k]}) and their corresponding bonds are retained. The
produced outputs are manipulated to update the MPS representation." SPEC.md:70-78 (truncated_svd_global)
fixes the contract this follows, with its design decisions: global ranking by value
descending, then charge ascending, then within-slice index ascending; values ≤ cutoff (1e−14) never kept.

Update (Vidal's canonical form, the MPS of PAPER.md:45; R21): Θ(c) = U_c diag(s_c) V_c†;
the kept values form the new λ^{[k]} (not renormalised: the factors reproduce the retained slices,
SPEC.md:74), each kept value carries its sector's charge c; the new bond is ordered by charge
ascending, then by value descending (a prefix of each sector's spectrum);
  Γ^{[k]}_new[α, a]   = U_c[α, s] / λ^{[k−1]}[α]     (α in Θ(c)'s rows; 0 elsewhere)
  Γ^{[k+1]}_new[a, β] = V_c†[s, β] / λ^{[k+1]}[β]    (β in Θ(c)'s columns; 0 elsewhere)
with a ↔ (c, s), and x/0 := 0. Rows/columns are returned in the CALLER's bond order.

Right-canonical ("B") form (Hastings, J. Math. Phys. 50, 095207 (2009); R22): an MPS stored as
B^{[k]} = Γ^{[k]} λ^{[k+1]} and λ's gives Θ(c) = λ^{[k−1]} B^{[k]} B^{[k+1]} (gated; tn_theta_exec with λk = λr = 1),
and the update needs no division by a singular value or a small λ:
  B^{[k]}_new[α, a]   = (Θ(c) V_c)[α, s] / λ^{[k−1]}[α]   (= Θ̃(c)·V_c, Θ̃ = Θ without its left λ; x/0 := 0)
  B^{[k+1]}_new[a, β] = V_c†[s, β]
(the division by λ^{[k−1]} undoes the row scaling Θ carries — each element to rounding — instead of dividing the
singular vectors U_c, whose absolute rounding errors the Vidal form amplifies by 1/λ).
"""
from __future__ import annotations

import numpy as np

from .theta import sector_ranges, sort_bonds


def sector_svds(sectors):
    """numpy SVD of every sector (library routine): list of (U, s, Vh), s descending."""
    out = []
    for th in sectors:
        if th.size == 0:
            out.append((np.zeros((th.shape[0], 0), complex), np.zeros(0), np.zeros((0, th.shape[1]), complex)))
        else:
            out.append(np.linalg.svd(th, full_matrices=False))
    return out


def global_top_chi(svals, chi_max: int, cutoff: float = 1e-14):
    """Global ranking: value desc, then charge asc, then index asc; keep ≤ chi_max values > cutoff.
    Returns (kept per sector k_c, discarded weight Σ dropped s²)."""
    entries = [(-float(v), c, i) for c, s in enumerate(svals) for i, v in enumerate(s)]
    entries.sort()
    kept = [0] * len(svals)
    disc = 0.0
    n = 0
    for negv, c, i in entries:
        v = -negv
        if n < chi_max and v > cutoff:
            kept[c] += 1
            n += 1
        else:
            disc += v * v
    return kept, disc


def truncate_update_rows(sectors, rows, cols, chi_l, chi_r, lam_l, lam_r, chi_max, cutoff=1e-14, form="vidal"):
    """The whole step on host for sectors given with their row / column bond lists: `rows[c]`, `cols[c]`
    are the CALLER indices of Θ(c)'s rows / columns (sector c = its position in `sectors`, which is the
    charge order of the ranking). Returns dict(chi, q_new (sector index per new bond), lam_new,
    gamma_k_new [χ_l × chi], gamma_k1_new [chi × χ_r], kept, discarded, svals). form="b": the right-canonical
    update of the module docstring (gamma_k_new = B^{[k]}_new, gamma_k1_new = B^{[k+1]}_new; lam_r unused)."""
    svd = sector_svds(sectors)
    kept, disc = global_top_chi([s for _, s, _ in svd], chi_max, cutoff)
    chi = sum(kept)
    gk = np.zeros((chi_l, chi), dtype=np.complex128)
    gk1 = np.zeros((chi, chi_r), dtype=np.complex128)
    q_new = np.zeros(chi, dtype=np.int32)
    lam_new = np.zeros(chi)
    a = 0
    for c in range(len(sectors)):
        k = kept[c]
        if k == 0:
            continue
        U, s, Vh = svd[c]
        ll = np.asarray(lam_l)[rows[c]]
        lr = np.asarray(lam_r)[cols[c]]
        inv_l = np.divide(1.0, ll, out=np.zeros_like(ll), where=ll != 0)
        inv_r = np.divide(1.0, lr, out=np.zeros_like(lr), where=lr != 0)
        if form == "b":
            gk[rows[c], a:a + k] = (sectors[c] @ Vh[:k, :].conj().T) * inv_l[:, None]
            gk1[a:a + k][:, cols[c]] = Vh[:k, :]
        else:
            gk[rows[c], a:a + k] = U[:, :k] * inv_l[:, None]
            gk1[a:a + k][:, cols[c]] = Vh[:k, :] * inv_r[None, :]
        q_new[a:a + k] = c
        lam_new[a:a + k] = s[:k]
        a += k
    return dict(chi=chi, q_new=q_new, lam_new=lam_new, gamma_k_new=gk, gamma_k1_new=gk1, kept=kept,
                discarded=disc, svals=[s for _, s, _ in svd])


def truncate_update(N, d, q_l, q_r, sectors, lam_l, lam_r, chi_max, cutoff=1e-14, form="vidal"):
    """Single-charge plans: Θ(c) rows are the sorted left bonds with c_l − c ∈ [0, d−1], columns the sorted
    right bonds with c − c_r ∈ [0, d−1] (oracle.theta.sector_ranges)."""
    perm_l, off_l = sort_bonds(q_l, N)
    perm_r, off_r = sort_bonds(q_r, N)
    rows, cols = [], []
    for c in range(N + 1):
        (r0, r1), (k0, k1) = sector_ranges(off_l, off_r, N, d, c)
        rows.append(perm_l[r0:r1])
        cols.append(perm_r[k0:k1])
    return truncate_update_rows(sectors, rows, cols, len(q_l), len(q_r), lam_l, lam_r, chi_max, cutoff, form)


def truncate_update2(N, d, q1_l, q2_l, q1_r, q2_r, sectors2, lam_l, lam_r, chi_max, cutoff=1e-14, form="vidal"):
    """MPO (pair-charge) plans: sector (c1, c2) has index c1·(N+1) + c2 — the ranking's
    charge order is the lexicographic pair order — and its rows / columns are the admissible
    sorted bonds of oracle.theta2 (l − c ∈ [0, d−1]², c − r ∈ [0, d−1]²). `sectors2[(c1, c2)]` as returned by
    oracle.theta2_sectors. Adds q1_new, q2_new (the kept values' charge pair)."""
    from .theta2 import pair_sector_cols, pair_sector_rows, sort_pair_bonds
    pl, pr = sort_pair_bonds(q1_l, q2_l), sort_pair_bonds(q1_r, q2_r)
    secs, rows, cols = [], [], []
    for c1 in range(N + 1):
        for c2 in range(N + 1):
            secs.append(sectors2[(c1, c2)])
            rows.append(pl[pair_sector_rows(np.asarray(q1_l)[pl], np.asarray(q2_l)[pl], d, c1, c2)])
            cols.append(pr[pair_sector_cols(np.asarray(q1_r)[pr], np.asarray(q2_r)[pr], d, c1, c2)])
    res = truncate_update_rows(secs, rows, cols, len(q1_l), len(q1_r), lam_l, lam_r, chi_max, cutoff, form)
    res["q1_new"], res["q2_new"] = np.divmod(res["q_new"], N + 1)
    return res
