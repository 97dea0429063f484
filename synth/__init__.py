"""Seeded synthetic inputs for the Θ(c) hot path — shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws bond charges, Γ tensors, λ
vectors and gate angles with the shapes and distributions of BASELINE.json configs 0–4
(recipe: SURVEY.md §8(d) "Generator"). The only structure it imposes is the input
sparsity pattern, i.e. Γ entries outside δ-allowed charge blocks are zero (SURVEY.md G4,
BASELINE.json config 0 "zero outside the allowed charge blocks").

Draw order per config (exactly, so per-seed counts are reproducible):
  1. charges q_l, q_c, q_r (in that order)
  2. Γk then Γk1: real parts then imaginary parts, (x + i y)/√2, masked
  3. λl, λk, λr
  4. θ, φ
  5. optional bond shuffle from default_rng(seed + 1000)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

__all__ = ["Case", "CONFIGS", "make_config", "make_case", "make_charges", "shuffle_case", "flat_lambda",
           "PairCase", "PAIR_CONFIGS", "make_pair_case", "make_pair_config", "vectorize_pure"]


@dataclass
class Case:
    """One two-site Θ problem. Arrays are in caller bond order (not necessarily sorted)."""
    name: str
    N: int
    d: int
    q_l: np.ndarray          # int32[chi_l]
    q_c: np.ndarray          # int32[chi_c]
    q_r: np.ndarray          # int32[chi_r]
    gamma_k: np.ndarray      # complex128[chi_l, chi_c]
    gamma_k1: np.ndarray     # complex128[chi_c, chi_r]
    lam_l: np.ndarray        # float64[chi_l]
    lam_k: np.ndarray        # float64[chi_c]
    lam_r: np.ndarray        # float64[chi_r]
    theta: float
    phi: float
    meta: dict = field(default_factory=dict)

    @property
    def chi_l(self) -> int:
        return int(self.q_l.shape[0])

    @property
    def chi_c(self) -> int:
        return int(self.q_c.shape[0])

    @property
    def chi_r(self) -> int:
        return int(self.q_r.shape[0])


# BASELINE.json configs 0..4: (N, d, chi, charge kind, lambda kind, seed)
CONFIGS = {
    0: dict(N=3, d=4, chi=16, charges="uniform", lam="random", seed=0, theta=0.7, phi=0.3),
    1: dict(N=7, d=8, chi=256, charges="uniform", lam="random", seed=1),
    2: dict(N=15, d=16, chi=1024, charges="gauss", lam="geometric", seed=2),
    3: dict(N=31, d=32, chi=4096, charges="gauss", lam="geometric", seed=3),
    4: dict(N=47, d=48, chi=8192, charges="gauss", lam="geometric", seed=4),
}


def _charges(rng, kind: str, N: int, chi: int) -> np.ndarray:
    if kind == "uniform":
        q = np.sort(rng.integers(0, N + 1, size=chi))
    elif kind == "gauss":
        # N(N/2, (N/4)^2), round to nearest, clip into [0, N], sort ascending.
        q = np.sort(np.clip(np.rint(rng.normal(N / 2, N / 4, size=chi)), 0, N))
    elif kind == "single":
        q = np.full(chi, int(rng.integers(0, N + 1)))
    else:
        raise ValueError(kind)
    return q.astype(np.int32)


def _gamma(rng, rows_q: np.ndarray, cols_q: np.ndarray, d: int) -> np.ndarray:
    shape = (rows_q.shape[0], cols_q.shape[0])
    g = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)
    diff = rows_q[:, None].astype(np.int64) - cols_q[None, :].astype(np.int64)
    g *= (diff >= 0) & (diff <= d - 1)
    return g


def _lam(rng, kind: str, chi: int) -> np.ndarray:
    if kind == "random":
        v = np.sort(1.0 - rng.random(chi))[::-1].copy()   # values in (0, 1], descending
    elif kind == "geometric":
        v = 0.995 ** np.arange(chi, dtype=np.float64)     # SURVEY.md G12 (no draws)
    elif kind == "steep":
        v = 0.97 ** np.arange(chi, dtype=np.float64)      # a wide Schmidt spectrum (no draws)
    elif kind == "flat":
        v = np.ones(chi)
    else:
        raise ValueError(kind)
    return v / np.linalg.norm(v)


def make_case(N: int, d: int, chi_l: int, chi_c: int, chi_r: int, seed, *, charges="uniform",
              lam="random", theta=None, phi=None, name="custom") -> Case:
    """Generic seeded case. `seed` is anything np.random.default_rng accepts."""
    rng = np.random.default_rng(seed)
    q_l = _charges(rng, charges, N, chi_l)
    q_c = _charges(rng, charges, N, chi_c)
    q_r = _charges(rng, charges, N, chi_r)
    gk = _gamma(rng, q_l, q_c, d)
    gk1 = _gamma(rng, q_c, q_r, d)
    lam_l = _lam(rng, lam, chi_l)
    lam_k = _lam(rng, lam, chi_c)
    lam_r = _lam(rng, lam, chi_r)
    if theta is None:
        theta = float(rng.uniform(0.0, math.pi / 2))
        phi = float(rng.uniform(0.0, 2 * math.pi))
    return Case(name, N, d, q_l, q_c, q_r, gk, gk1, lam_l, lam_k, lam_r, float(theta), float(phi),
                meta=dict(seed=seed if isinstance(seed, int) else list(seed), charges=charges, lam=lam))


def make_charges(cfg: int, gate: int = 0, shuffled: bool = False):
    """Only step 1 of make_config (identical draws): (N, d, q_l, q_c, q_r) without building Γ."""
    c = CONFIGS[cfg]
    rng = np.random.default_rng([4, gate] if cfg == 4 else c["seed"])
    qs = [_charges(rng, c["charges"], c["N"], c["chi"]) for _ in range(3)]
    if shuffled:
        rng2 = np.random.default_rng(c["seed"] + 1000)
        qs = [np.ascontiguousarray(q[rng2.permutation(c["chi"])]) for q in qs]
    return c["N"], c["d"], qs[0], qs[1], qs[2]


def make_config(cfg: int, gate: int = 0, *, shuffled: bool = False, flat: bool = False) -> Case:
    """BASELINE.json config `cfg` (0..4). Config 4 gate g draws from default_rng([4, g])."""
    c = CONFIGS[cfg]
    seed = [4, gate] if cfg == 4 else c["seed"]
    case = make_case(c["N"], c["d"], c["chi"], c["chi"], c["chi"], seed, charges=c["charges"],
                     lam=c["lam"], theta=c.get("theta"), phi=c.get("phi"), name=f"config{cfg}")
    case.meta["config"] = cfg
    case.meta["gate"] = gate
    if shuffled:
        case = shuffle_case(case, c["seed"] + 1000)
    if flat:
        case = flat_lambda(case)
    return case


def shuffle_case(case: Case, seed) -> Case:
    """Apply one random permutation per bond consistently to q, the matching Γ axis and λ."""
    rng2 = np.random.default_rng(seed)
    pl = rng2.permutation(case.chi_l)
    pc = rng2.permutation(case.chi_c)
    pr = rng2.permutation(case.chi_r)
    return replace(case, name=case.name + "-shuffled",
                   q_l=np.ascontiguousarray(case.q_l[pl]), q_c=np.ascontiguousarray(case.q_c[pc]),
                   q_r=np.ascontiguousarray(case.q_r[pr]),
                   gamma_k=np.ascontiguousarray(case.gamma_k[pl][:, pc]),
                   gamma_k1=np.ascontiguousarray(case.gamma_k1[pc][:, pr]),
                   lam_l=np.ascontiguousarray(case.lam_l[pl]), lam_k=np.ascontiguousarray(case.lam_k[pc]),
                   lam_r=np.ascontiguousarray(case.lam_r[pr]),
                   meta=dict(case.meta, shuffled=True))


def flat_lambda(case: Case) -> Case:
    """SURVEY.md G12 flat-λ variant: λl = λk = λr = 1/√χ, everything else identical."""
    return replace(case, name=case.name + "-flat",
                   lam_l=np.full(case.chi_l, 1 / math.sqrt(case.chi_l)),
                   lam_k=np.full(case.chi_c, 1 / math.sqrt(case.chi_c)),
                   lam_r=np.full(case.chi_r, 1 / math.sqrt(case.chi_r)),
                   meta=dict(case.meta, flat=True))


# ---------------------------------------------------------------------------------------------
# MPO (doubled-charge) inputs: each bond carries a charge pair (c1, c2). No
# BASELINE.json config covers this path; PAIR_CONFIGS are shaped like the paper's MPO GPU runs
# (N = 5 photons, d = N + 1, PAPER.md:192/:207 use χ = 4096) — DESIGN.md §3.
# ---------------------------------------------------------------------------------------------
@dataclass
class PairCase:
    name: str
    N: int
    d: int
    q1_l: np.ndarray
    q2_l: np.ndarray
    q1_c: np.ndarray
    q2_c: np.ndarray
    q1_r: np.ndarray
    q2_r: np.ndarray
    gamma_k: np.ndarray
    gamma_k1: np.ndarray
    lam_l: np.ndarray
    lam_k: np.ndarray
    lam_r: np.ndarray
    theta: float
    phi: float
    meta: dict = field(default_factory=dict)

    @property
    def chi_l(self) -> int:
        return int(self.q1_l.shape[0])

    @property
    def chi_c(self) -> int:
        return int(self.q1_c.shape[0])

    @property
    def chi_r(self) -> int:
        return int(self.q1_r.shape[0])


PAIR_CONFIGS = {
    0: dict(N=2, d=3, chi=24, charges="uniform", lam="random", seed=100, theta=0.7, phi=0.3),
    1: dict(N=4, d=5, chi=256, charges="uniform", lam="random", seed=101),
    2: dict(N=5, d=6, chi=1024, charges="gauss", lam="geometric", seed=102),
    3: dict(N=5, d=6, chi=4096, charges="gauss", lam="geometric", seed=103),
    # the paper's larger MPO charge ranges: d = 14 (Fig. S2(b)) and d = 18 (its largest run,
    # PAPER.md:408), with N = d − 1 so every occupation 0..d−1 is reachable; (N+1)² = 196 / 324 pair keys
    4: dict(N=13, d=14, chi=4096, charges="gauss", lam="geometric", seed=104),
    5: dict(N=17, d=18, chi=4096, charges="gauss", lam="geometric", seed=105),
}


def _pair_charges(rng, kind, N, chi):
    """Two charge components per bond, drawn independently, then ordered lexicographically."""
    a = _charges(rng, kind, N, chi)
    b = _charges(rng, kind, N, chi)
    b = b[rng.permutation(chi)]          # decorrelate the sorted second component
    o = np.lexsort((b, a))
    return a[o].astype(np.int32), b[o].astype(np.int32)


def _pair_gamma(rng, r1, r2, c1, c2, d):
    shape = (r1.shape[0], c1.shape[0])
    g = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)
    for a, b in ((r1, c1), (r2, c2)):
        diff = a[:, None].astype(np.int64) - b[None, :].astype(np.int64)
        g *= (diff >= 0) & (diff <= d - 1)
    return g


def make_pair_case(N, d, chi_l, chi_c, chi_r, seed, *, charges="uniform", lam="random", theta=None, phi=None,
                   name="pair") -> PairCase:
    rng = np.random.default_rng(seed)
    q1_l, q2_l = _pair_charges(rng, charges, N, chi_l)
    q1_c, q2_c = _pair_charges(rng, charges, N, chi_c)
    q1_r, q2_r = _pair_charges(rng, charges, N, chi_r)
    gk = _pair_gamma(rng, q1_l, q2_l, q1_c, q2_c, d)
    gk1 = _pair_gamma(rng, q1_c, q2_c, q1_r, q2_r, d)
    lam_l, lam_k, lam_r = _lam(rng, lam, chi_l), _lam(rng, lam, chi_c), _lam(rng, lam, chi_r)
    if theta is None:
        theta = float(rng.uniform(0.0, math.pi / 2))
        phi = float(rng.uniform(0.0, 2 * math.pi))
    return PairCase(name, N, d, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r, gk, gk1, lam_l, lam_k, lam_r, float(theta),
                    float(phi), meta=dict(seed=seed, charges=charges, lam=lam))


def make_pair_config(cfg: int) -> PairCase:
    c = PAIR_CONFIGS[cfg]
    return make_pair_case(c["N"], c["d"], c["chi"], c["chi"], c["chi"], c["seed"], charges=c["charges"],
                          lam=c["lam"], theta=c.get("theta"), phi=c.get("phi"), name=f"pair{cfg}")


def vectorize_pure(case: Case) -> PairCase:
    """The vectorized pure state |ψ⟩⟨ψ| of a single-charge case: bond (α, α') with charges
    (q[α], q[α']), Γ2[(α,α'),(β,β')] = Γ[α,β]·conj(Γ[α',β']), λ2 = λ[α]λ[α'] (row-major pair index)."""
    def pairq(q):
        return np.repeat(q, q.shape[0]).astype(np.int32), np.tile(q, q.shape[0]).astype(np.int32)
    q1_l, q2_l = pairq(case.q_l)
    q1_c, q2_c = pairq(case.q_c)
    q1_r, q2_r = pairq(case.q_r)
    gk = np.kron(case.gamma_k, np.conj(case.gamma_k))
    gk1 = np.kron(case.gamma_k1, np.conj(case.gamma_k1))
    return PairCase(case.name + "-vectorized", case.N, case.d, q1_l, q2_l, q1_c, q2_c, q1_r, q2_r, gk, gk1,
                    np.kron(case.lam_l, case.lam_l), np.kron(case.lam_k, case.lam_k), np.kron(case.lam_r, case.lam_r),
                    case.theta, case.phi, meta=dict(vectorized=case.name))
