"""Brick-wall layers of beam-splitter gates on a device-resident U(1) MPS.

Host orchestration only (argument marshalling): every gate is tn_theta_plan (K1) → tn_build_bs_unitary
(K2) → tn_theta_exec (K3–K5) → tn_svd_truncate_bform (per-sector SVD + global top-χ + right-canonical update),
all in libtn_theta.so. The MPS is the canonical form of PAPER.md:45 with the U(1) constraint of
PAPER.md:49-51, kept in right-canonical ("B") form: site k carries B^{[k]} = Γ^{[k]}λ^{[k+1]} [χ_k × χ_{k+1}]
(complex128, rows/columns in the bonds' stored order), bond k carries λ (float64) and its charges (int32,
photons to the right); bond 0 is one bond of charge N, bond M one bond of charge 0. A gate on sites (k, k+1)
builds Θ(c) = λ^{[k]} B^{[k]} B^{[k+1]} (gated; Eq. S5 with the inner λ's inside the B's) and replaces B^{[k]},
λ^{[k+1]}, q^{[k+1]}, B^{[k+1]} without dividing by any singular value or small λ (Hastings' update, DESIGN.md
R22; oracle: oracle/layer.py with form "b"). Vidal states (Γ, λ) are converted on construction (B = Γλ).

Layer parallelism ("beam splitter updates within a layer are parallel"; PAPER.md:96-103
first-level parallelism): with a torch.distributed process group, every rank holds a replica of the MPS,
the gates of a layer (disjoint site pairs, so independent) are dealt to ranks by longest-processing-time
on their Θ flop estimate (χ_k·χ_{k+1}·χ_{k+2}, identical on every rank), each rank runs its own gates
on its GPU, and the owner of each gate broadcasts the four updated tensors (NCCL over NVLink; ~0.3 ms
per config-3 Γ at 900 GB/s against ~0.35 s of SVD per gate), so every replica ends the layer identical.
"""
from __future__ import annotations

import numpy as np
import torch

from . import Plan, Plan2, build_bs_unitary, svd_truncate, theta_exec


def layer_owners(costs, world: int):
    """Longest-processing-time assignment of independent gates to `world` ranks: gates in decreasing
    cost (ties: lower gate index first) each go to the currently least-loaded rank (ties: lower rank).
    Deterministic, so every rank computes the same table without communication."""
    order = sorted(range(len(costs)), key=lambda g: (-costs[g], g))
    load = [0.0] * world
    owner = [0] * len(costs)
    for g in order:
        r = min(range(world), key=lambda x: (load[x], x))
        owner[g] = r
        load[r] += costs[g]
    return owner


class _Chain:
    """Layer logic shared by MPS and MPO: `_charges()` lists the per-bond charge lists (one species for an
    MPS, two for an MPO), `apply_gate` updates sites (k, k+1)."""

    def _charges(self):
        raise NotImplementedError

    def gate_cost(self, k: int) -> float:
        """Θ-build flop estimate of the gate on (k, k+1) used to balance a layer: χ_k·χ_{k+1}·χ_{k+2}."""
        q = self._charges()[0]
        return float(q[k].numel()) * float(q[k + 1].numel()) * float(q[k + 2].numel())

    def apply_layer(self, parity: int, thetas, phis, chi_max: int, cutoff: float = 1e-14, contraction=None,
                    group=None):
        """Gates on (k, k+1) for k = parity, parity+2, … < M−1; returns their discarded weights.

        With `group` (a torch.distributed process group of size > 1) the gates are spread over its ranks
        (layer_owners) and the results broadcast, leaving every rank's replica identical."""
        ks = list(range(parity, self.M - 1, 2))
        world = 1
        if group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(group)
        if world == 1:
            return [self.apply_gate(k, thetas[g], phis[g], chi_max, cutoff, contraction) for g, k in enumerate(ks)]
        import torch.distributed as dist
        me = dist.get_rank(group)
        owner = layer_owners([self.gate_cost(k) for k in ks], world)
        disc = torch.zeros(len(ks), dtype=torch.float64, device=self.device)
        for g, k in enumerate(ks):
            if owner[g] == me:
                disc[g] = float(self.apply_gate(k, thetas[g], phis[g], chi_max, cutoff, contraction))
        for g, k in enumerate(ks):   # every rank walks the gates in the same order
            self._bcast_gate(k, owner[g], owner[g] == me, group)
        dist.all_reduce(disc, group=group)   # each entry has exactly one non-zero contributor
        return [float(x) for x in disc.cpu()]

    def _bcast_gate(self, k: int, src: int, mine: bool, group):
        """Broadcast the tensors gate (k, k+1) replaced — the charges of bond k+1 (every species), λ^{[k+1]},
        Γ^{[k]}, Γ^{[k+1]} — from group rank `src`."""
        import torch.distributed as dist
        dev = self.device
        qs = self._charges()
        bc = lambda t: dist.broadcast(t, group=group, group_src=src)
        if mine:  # the owner's freshly written tensors are sent as they are (contiguous)
            self.gam[k], self.gam[k + 1] = self.gam[k].contiguous(), self.gam[k + 1].contiguous()
            self.lam[k + 1] = self.lam[k + 1].contiguous()
        n = torch.tensor([qs[0][k + 1].numel() if mine else 0], dtype=torch.int64, device=dev)
        bc(n)
        chi = int(n.item())
        chi_l, chi_r = qs[0][k].numel(), qs[0][k + 2].numel()
        if not mine:
            for q in qs:
                q[k + 1] = torch.empty(chi, dtype=torch.int32, device=dev)
            self.lam[k + 1] = torch.empty(chi, dtype=torch.float64, device=dev)
            self.gam[k] = torch.empty((chi_l, chi), dtype=torch.complex128, device=dev)
            self.gam[k + 1] = torch.empty((chi, chi_r), dtype=torch.complex128, device=dev)
        if chi == 0:
            return
        for q in qs:
            q64 = q[k + 1].to(torch.int64)   # int32 broadcast is not available on every backend
            bc(q64)
            if not mine:
                q[k + 1] = q64.to(torch.int32)
        bc(self.lam[k + 1])
        for t in (self.gam[k], self.gam[k + 1]):
            if t.numel():
                bc(torch.view_as_real(t))


def _to_b(gam, lam, form):
    """Site tensors in right-canonical form: B^{[k]} = Γ^{[k]}λ^{[k+1]} for a Vidal input (a product, no division)."""
    if form == "b":
        return gam
    return [(g * l[None, :]).contiguous() for g, l in zip(gam, lam[1:])]


class MPS(_Chain):
    def __init__(self, N: int, d: int, q, gam, lam, device="cuda", form: str = "vidal"):
        """`gam`: Vidal Γ^{[k]} (form "vidal", converted) or right-canonical B^{[k]} (form "b")."""
        dev = torch.device(device)
        as_t = lambda x, dt: (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))).to(
            dev, dt).contiguous()
        self.N, self.d = int(N), int(d)
        self.device = dev
        self.q = [as_t(x, torch.int32) for x in q]
        self.lam = [as_t(x, torch.float64) for x in lam]
        self.gam = _to_b([as_t(x, torch.complex128) for x in gam], self.lam, form)   # B^{[k]}
        self.M = len(self.gam)
        if len(self.q) != self.M + 1 or len(self.lam) != self.M + 1:
            raise ValueError("an MPS of M sites needs M+1 bonds of charges and λ")

    @classmethod
    def from_state(cls, st: dict, device="cuda"):
        return cls(st["N"], st["d"], st["q"], st["gam"], st["lam"], device, st.get("form", "vidal"))

    def to_state(self) -> dict:
        """Host copy in right-canonical form (oracle/layer.py state dict with form "b")."""
        return dict(N=self.N, d=self.d, q=[x.cpu().numpy() for x in self.q], gam=[x.cpu().numpy() for x in self.gam],
                    lam=[x.cpu().numpy() for x in self.lam], form="b")

    def _ones(self, n: int):
        return torch.ones(n, dtype=torch.float64, device=self.device)

    def apply_gate(self, k: int, theta: float, phi: float, chi_max: int, cutoff: float = 1e-14, contraction=None):
        """One TEBD update of sites (k, k+1); returns the discarded weight Σ dropped s²."""
        if not 0 <= k < self.M - 1:
            raise ValueError("gate sites out of range")
        plan = Plan(self.d, self.N, self.q[k], self.q[k + 1], self.q[k + 2])
        if contraction is not None:
            plan.set_contraction(*contraction)
        U = build_bs_unitary(plan, theta, phi)
        # Θ = λ^{[k]} B^{[k]} B^{[k+1]} (gated): the inner λ's are inside the B's
        out = theta_exec(plan, self.gam[k], self._ones(plan.chi[1]), self.gam[k + 1], self.lam[k],
                         self._ones(plan.chi[2]), U)
        res = svd_truncate(plan, out, self.lam[k], None, chi_max, cutoff, form="b")
        self.q[k + 1] = res["q_new"]
        self.lam[k + 1] = res["lam_new"]
        self.gam[k] = res["gamma_k_new"]
        self.gam[k + 1] = res["gamma_k1_new"]
        plan.destroy()
        return res["discarded"]

    def _charges(self):
        return [self.q]


class MPO(_Chain):
    """A vectorized density matrix on the device ("MPOs are vectorized into the MPS
    form, U → U⊗U*, and two conserved charges are present"): bond k carries charge PAIRS (q1, q2) (ket, bra
    photons to the right, int32 each), λ (float64); site k carries Γ^{[k]} [χ_k × χ_{k+1}] complex128. A gate
    on sites (k, k+1) is tn_theta2_plan → U → tn_theta_exec (Θ(c1, c2), two-pass U⊗U* mix) →
    tn_svd_truncate on the pair plan (oracle: oracle/layer.py apply_gate2)."""

    def __init__(self, N: int, d: int, q1, q2, gam, lam, device="cuda", form: str = "vidal"):
        dev = torch.device(device)
        as_t = lambda x, dt: (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))).to(
            dev, dt).contiguous()
        self.N, self.d, self.device = int(N), int(d), dev
        self.q1 = [as_t(x, torch.int32) for x in q1]
        self.q2 = [as_t(x, torch.int32) for x in q2]
        self.lam = [as_t(x, torch.float64) for x in lam]
        self.gam = _to_b([as_t(x, torch.complex128) for x in gam], self.lam, form)   # B^{[k]}
        self.M = len(self.gam)
        if not (len(self.q1) == len(self.q2) == len(self.lam) == self.M + 1):
            raise ValueError("an MPO of M sites needs M+1 bonds of charge pairs and λ")

    @classmethod
    def from_state(cls, st: dict, device="cuda"):
        return cls(st["N"], st["d"], st["q1"], st["q2"], st["gam"], st["lam"], device, st.get("form", "vidal"))

    def to_state(self) -> dict:
        c = lambda xs: [x.cpu().numpy() for x in xs]
        return dict(N=self.N, d=self.d, q1=c(self.q1), q2=c(self.q2), gam=c(self.gam), lam=c(self.lam), form="b")

    def _ones(self, n: int):
        return torch.ones(n, dtype=torch.float64, device=self.device)

    def apply_gate(self, k: int, theta: float, phi: float, chi_max: int, cutoff: float = 1e-14, contraction=None):
        """One TEBD update of sites (k, k+1) with U⊗U*; returns the discarded weight."""
        if not 0 <= k < self.M - 1:
            raise ValueError("gate sites out of range")
        plan = Plan2(self.d, self.N, self.q1[k], self.q2[k], self.q1[k + 1], self.q2[k + 1], self.q1[k + 2],
                     self.q2[k + 2])
        if contraction is not None:
            plan.set_contraction(*contraction)
        U = build_bs_unitary(plan, theta, phi)
        out = theta_exec(plan, self.gam[k], self._ones(plan.chi[1]), self.gam[k + 1], self.lam[k],
                         self._ones(plan.chi[2]), U)
        res = svd_truncate(plan, out, self.lam[k], None, chi_max, cutoff, form="b")
        self.q1[k + 1] = res["q1_new"].to(torch.int32).contiguous()
        self.q2[k + 1] = res["q2_new"].to(torch.int32).contiguous()
        self.lam[k + 1] = res["lam_new"]
        self.gam[k] = res["gamma_k_new"]
        self.gam[k + 1] = res["gamma_k1_new"]
        plan.destroy()
        return res["discarded"]

    def _charges(self):
        return [self.q1, self.q2]
