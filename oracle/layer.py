"""Plain CPU oracle of a brick-wall layer of beam-splitter gates on a U(1) MPS (TEST INFRASTRUCTURE ONLY).

SURVEY.md §8(f) NEXT-3, BASELINE.json config 4 ("a brick-wall layer of beam-splitter gates on an M-mode
MPS"), PAPER.md:99 ("beam splitter updates within a layer are parallel"). The MPS is the Vidal form of
PAPER.md:45 with the U(1) constraint of PAPER.md:49-51: sites 0..M−1 carry Γ^{[k]} [χ_k × χ_{k+1}] (the
physical index i_k = c(α_k) − c(α_{k+1}) is implied by the bond charges), bonds 0..M carry λ and charges
(bond 0: one bond of charge N; bond M: one bond of charge 0). A gate on sites (k, k+1) is Eq. S5's Θ
(oracle.theta_sectors with left/centre/right bonds k, k+1, k+2) followed by the SVD update
(oracle.svd.truncate_update); gates of one layer act on disjoint site pairs.
"""
from __future__ import annotations

import itertools

import numpy as np

from .svd import truncate_update
from .theta import theta_sectors


def _form(state):
    return state.get("form", "vidal")


def _inner(state, k):
    """The λ's Θ of Eq. S5 puts between / right of the two sites: Vidal form uses the stored λ^{[k+1]}, λ^{[k+2]};
    the right-canonical form (gam holds B^{[k]} = Γ^{[k]}λ^{[k+1]}, oracle/svd.py) has them inside its B's."""
    lam = state["lam"]
    if _form(state) == "b":
        return np.ones(len(lam[k + 1])), np.ones(len(lam[k + 2]))
    return lam[k + 1], lam[k + 2]


def to_bform(state):
    """Vidal → right-canonical form: B^{[k]} = Γ^{[k]} λ^{[k+1]} (a product, no division)."""
    out = {key: ([x.copy() for x in v] if isinstance(v, list) else v) for key, v in state.items()}
    out["gam"] = [g * state["lam"][k + 1][None, :] for k, g in enumerate(state["gam"])]
    out["form"] = "b"
    return out


def apply_gate(state, k, theta, phi, chi_max, cutoff=1e-14):
    """In-place TEBD update of sites (k, k+1). `state` = dict(N, d, q: [M+1 int arrays], gam: [M complex],
    lam: [M+1 real], optional form: "vidal" (default) | "b" (gam holds B^{[k]}, the update of oracle/svd.py's
    right-canonical form)). Returns the discarded weight."""
    N, d = state["N"], state["d"]
    q, gam, lam = state["q"], state["gam"], state["lam"]
    lk, lr = _inner(state, k)
    secs, *_ = theta_sectors(N, d, q[k], q[k + 1], q[k + 2], gam[k], lk, gam[k + 1], lam[k], lr, theta, phi)
    res = truncate_update(N, d, q[k], q[k + 2], secs, lam[k], lr, chi_max, cutoff, _form(state))
    q[k + 1] = res["q_new"]
    lam[k + 1] = res["lam_new"]
    gam[k] = res["gamma_k_new"]
    gam[k + 1] = res["gamma_k1_new"]
    return res["discarded"]


def apply_layer(state, parity, thetas, phis, chi_max, cutoff=1e-14):
    """Gates on (k, k+1) for k = parity, parity+2, … < M−1, in increasing k (they commute)."""
    M = len(state["gam"])
    disc = []
    for g, k in enumerate(range(parity, M - 1, 2)):
        disc.append(apply_gate(state, k, thetas[g], phis[g], chi_max, cutoff))
    return disc


def dense_state(state):
    """c[i_0, …, i_{M−1}] = Σ Γ^{[0]} λ^{[1]} Γ^{[1]} … Γ^{[M−1]} with the outer λ's (bond 0 and M) and the δ's
    (i_k = c(α_k) − c(α_{k+1}) ∈ [0, d−1]) written out — small M only."""
    N, d = state["N"], state["d"]
    q, gam, lam = state["q"], state["gam"], state["lam"]
    M = len(gam)
    # vec[α_k, i_0..i_{k−1}]
    vec = np.asarray(lam[0], dtype=np.complex128).copy()
    for k in range(M):
        G = gam[k] if _form(state) == "b" else gam[k] * lam[k + 1][None, :]
        new = np.zeros((len(q[k + 1]),) + (d,) * (k + 1), dtype=np.complex128)
        for a in range(len(q[k])):
            for b in range(len(q[k + 1])):
                i = int(q[k][a]) - int(q[k + 1][b])
                if 0 <= i <= d - 1 and G[a, b] != 0:
                    new[(b,) + (slice(None),) * k + (i,)] += vec[a] * G[a, b]
        vec = new
    return vec.sum(axis=0)     # the single right boundary bond


def dense_gate(psi, k, U4):
    """Apply ⟨i,i'|U|j,j'⟩ (U4[i, i', j, j']) to modes (k, k+1) of a dense state."""
    M = psi.ndim
    perm = [k, k + 1] + [m for m in range(M) if m not in (k, k + 1)]
    x = np.transpose(psi, perm)
    sh = x.shape
    x = np.einsum("abij,ij...->ab...", U4, x.reshape(sh))
    return np.transpose(x, np.argsort(perm))


def random_mps(M, N, d, chi, seed):
    """A random U(1) MPS with valid charges: bond k's charges lie in the reachable window
    [max(0, N − k(d−1)), min(N, (M−k)(d−1))] (photons to the right), sorted; Γ masked to allowed blocks."""
    rng = np.random.default_rng(seed)
    q = []
    for k in range(M + 1):
        if k == 0:
            q.append(np.array([N], dtype=np.int32))
        elif k == M:
            q.append(np.array([0], dtype=np.int32))
        else:
            lo, hi = max(0, N - k * (d - 1)), min(N, (M - k) * (d - 1))
            q.append(np.sort(rng.integers(lo, hi + 1, size=chi)).astype(np.int32))
    gam = []
    for k in range(M):
        a, b = q[k], q[k + 1]
        g = (rng.standard_normal((len(a), len(b))) + 1j * rng.standard_normal((len(a), len(b)))) / np.sqrt(2)
        diff = a[:, None].astype(np.int64) - b[None, :]
        gam.append(g * ((diff >= 0) & (diff <= d - 1)))
    lam = [np.ones(1)] + [np.sort(rng.uniform(0.2, 1.0, size=len(q[k])))[::-1].copy() for k in range(1, M)] + [np.ones(1)]
    return dict(N=N, d=d, q=q, gam=gam, lam=lam)


def copy_state(s):
    return dict(N=s["N"], d=s["d"], q=[x.copy() for x in s["q"]], gam=[x.copy() for x in s["gam"]],
                lam=[x.copy() for x in s["lam"]], form=_form(s))


# ---------------------------------------------------------------------------------------------------------
# MPO (vectorized density matrix, two conserved charges) — PAPER.md:101, :105-107: "MPOs are vectorized into
# the MPS form, U → U⊗U*, and two conserved charges are present". Bond k carries charge PAIRS (q1, q2) (ket,
# bra photons to the right); site k's physical pair (i, i') is implied by i = q1_k − q1_{k+1}, i' = q2_k − q2_{k+1}.
# A gate is Θ(c1, c2) (oracle.theta2_sectors) followed by the pair SVD update (oracle.svd.truncate_update2).
# ---------------------------------------------------------------------------------------------------------
def apply_gate2(state, k, theta, phi, chi_max, cutoff=1e-14):
    """In-place TEBD update of MPO sites (k, k+1). `state` = dict(N, d, q1, q2: [M+1 int arrays], gam: [M],
    lam: [M+1]). Returns the discarded weight."""
    from .svd import truncate_update2
    from .theta2 import theta2_sectors
    N, d = state["N"], state["d"]
    q1, q2, gam, lam = state["q1"], state["q2"], state["gam"], state["lam"]
    lk, lr = _inner(state, k)
    secs, *_ = theta2_sectors(N, d, q1[k], q2[k], q1[k + 1], q2[k + 1], q1[k + 2], q2[k + 2], gam[k], lk,
                              gam[k + 1], lam[k], lr, theta, phi)
    res = truncate_update2(N, d, q1[k], q2[k], q1[k + 2], q2[k + 2], secs, lam[k], lr, chi_max, cutoff,
                           _form(state))
    q1[k + 1], q2[k + 1] = res["q1_new"].astype(np.int32), res["q2_new"].astype(np.int32)
    lam[k + 1] = res["lam_new"]
    gam[k] = res["gamma_k_new"]
    gam[k + 1] = res["gamma_k1_new"]
    return res["discarded"]


def apply_layer2(state, parity, thetas, phis, chi_max, cutoff=1e-14):
    M = len(state["gam"])
    return [apply_gate2(state, k, thetas[g], phis[g], chi_max, cutoff) for g, k in enumerate(range(parity, M - 1, 2))]


def vectorize_mps(state):
    """|ψ⟩⟨ψ| of a Vidal MPS as a vectorized MPO: pair bond (α, α') with charges (q[α], q[α']),
    Γ2 = Γ ⊗ conj(Γ), λ2 = λ ⊗ λ (row-major pair index)."""
    pq = lambda q: (np.repeat(q, len(q)).astype(np.int32), np.tile(q, len(q)).astype(np.int32))
    q1, q2 = zip(*(pq(q) for q in state["q"]))
    return dict(N=state["N"], d=state["d"], q1=list(q1), q2=list(q2),
                gam=[np.kron(g, np.conj(g)) for g in state["gam"]], lam=[np.kron(l, l) for l in state["lam"]],
                form=_form(state))


def dense_state2(state):
    """ρ[i_0..i_{M−1}, i'_0..i'_{M−1}] of a small vectorized MPO: the chain contracted like dense_state with
    the physical pair (i, i') = (q1_k − q1_{k+1}, q2_k − q2_{k+1}) ∈ [0, d−1]² (both δ's written out)."""
    N, d = state["N"], state["d"]
    q1, q2, gam, lam = state["q1"], state["q2"], state["gam"], state["lam"]
    M = len(gam)
    vec = np.asarray(lam[0], dtype=np.complex128).copy()
    for k in range(M):
        G = gam[k] if _form(state) == "b" else gam[k] * lam[k + 1][None, :]
        new = np.zeros((len(q1[k + 1]),) + (d * d,) * (k + 1), dtype=np.complex128)
        for a in range(len(q1[k])):
            for b in range(len(q1[k + 1])):
                i, ip = int(q1[k][a]) - int(q1[k + 1][b]), int(q2[k][a]) - int(q2[k + 1][b])
                if 0 <= i <= d - 1 and 0 <= ip <= d - 1 and G[a, b] != 0:
                    new[(b,) + (slice(None),) * k + (i * d + ip,)] += vec[a] * G[a, b]
        vec = new
    x = vec.sum(axis=0).reshape((d, d) * M)              # axes (i_0, i'_0, i_1, i'_1, …)
    return np.transpose(x, list(range(0, 2 * M, 2)) + list(range(1, 2 * M, 2)))


def random_mpo(M, N, d, chi, seed):
    """A random vectorized-MPO-shaped state with two independent charge species per bond (each in the
    reachable window of random_mps), Γ masked to blocks allowed for BOTH species; bonds sorted by pair key."""
    rng = np.random.default_rng(seed)
    q1, q2 = [], []
    for k in range(M + 1):
        if k == 0:
            a = b = np.array([N], dtype=np.int32)
        elif k == M:
            a = b = np.array([0], dtype=np.int32)
        else:
            lo, hi = max(0, N - k * (d - 1)), min(N, (M - k) * (d - 1))
            a = rng.integers(lo, hi + 1, size=chi)
            b = rng.integers(lo, hi + 1, size=chi)
            o = np.lexsort((b, a))
            a, b = a[o].astype(np.int32), b[o].astype(np.int32)
        q1.append(a)
        q2.append(b)
    gam = []
    for k in range(M):
        g = (rng.standard_normal((len(q1[k]), len(q1[k + 1]))) + 1j * rng.standard_normal((len(q1[k]), len(q1[k + 1])))) / np.sqrt(2)
        d1 = q1[k][:, None].astype(np.int64) - q1[k + 1][None, :]
        d2 = q2[k][:, None].astype(np.int64) - q2[k + 1][None, :]
        gam.append(g * ((d1 >= 0) & (d1 <= d - 1) & (d2 >= 0) & (d2 <= d - 1)))
    lam = [np.ones(1)] + [np.sort(rng.uniform(0.2, 1.0, size=len(q1[k])))[::-1].copy() for k in range(1, M)] + [np.ones(1)]
    return dict(N=N, d=d, q1=q1, q2=q2, gam=gam, lam=lam)


def copy_state2(s):
    return dict(N=s["N"], d=s["d"], q1=[x.copy() for x in s["q1"]], q2=[x.copy() for x in s["q2"]],
                gam=[x.copy() for x in s["gam"]], lam=[x.copy() for x in s["lam"]], form=_form(s))
