"""Brick-wall layers of beam-splitter gates on a device-resident U(1) MPS.

Host orchestration only (argument marshalling): every gate is tn_theta_plan (K1) → tn_build_bs_unitary
(K2) → tn_theta_exec (K3–K5) → tn_svd_truncate (per-sector SVD + global top-χ + Vidal update), all in
libtn_theta.so. The MPS is the Vidal form of PAPER.md:45 with the U(1) constraint of PAPER.md:49-51:
site k carries Γ^{[k]} [χ_k × χ_{k+1}] (complex128, rows/columns in the bonds' stored order), bond k
carries λ (float64) and its charges (int32, photons to the right); bond 0 is one bond of charge N,
bond M one bond of charge 0. A gate on sites (k, k+1) uses bonds k, k+1, k+2 as the left, centre and
right bonds of Eq. S5 and replaces Γ^{[k]}, λ^{[k+1]}, q^{[k+1]}, Γ^{[k+1]} (oracle: oracle/layer.py).
Gates of one layer act on disjoint site pairs ("beam splitter updates within a layer are
parallel"); here they run one after another on the current device.
"""
from __future__ import annotations

import numpy as np
import torch

from . import Plan, build_bs_unitary, svd_truncate, theta_exec


class MPS:
    def __init__(self, N: int, d: int, q, gam, lam, device="cuda"):
        dev = torch.device(device)
        as_t = lambda x, dt: (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))).to(
            dev, dt).contiguous()
        self.N, self.d = int(N), int(d)
        self.q = [as_t(x, torch.int32) for x in q]
        self.gam = [as_t(x, torch.complex128) for x in gam]
        self.lam = [as_t(x, torch.float64) for x in lam]
        self.M = len(self.gam)
        if len(self.q) != self.M + 1 or len(self.lam) != self.M + 1:
            raise ValueError("an MPS of M sites needs M+1 bonds of charges and λ")

    @classmethod
    def from_state(cls, st: dict, device="cuda"):
        return cls(st["N"], st["d"], st["q"], st["gam"], st["lam"], device)

    def to_state(self) -> dict:
        return dict(N=self.N, d=self.d, q=[x.cpu().numpy() for x in self.q], gam=[x.cpu().numpy() for x in self.gam],
                    lam=[x.cpu().numpy() for x in self.lam])

    def apply_gate(self, k: int, theta: float, phi: float, chi_max: int, cutoff: float = 1e-14, contraction=None):
        """One TEBD update of sites (k, k+1); returns the discarded weight Σ dropped s²."""
        if not 0 <= k < self.M - 1:
            raise ValueError("gate sites out of range")
        plan = Plan(self.d, self.N, self.q[k], self.q[k + 1], self.q[k + 2])
        if contraction is not None:
            plan.set_contraction(*contraction)
        U = build_bs_unitary(plan, theta, phi)
        out = theta_exec(plan, self.gam[k], self.lam[k + 1], self.gam[k + 1], self.lam[k], self.lam[k + 2], U)
        res = svd_truncate(plan, out, self.lam[k], self.lam[k + 2], chi_max, cutoff)
        self.q[k + 1] = res["q_new"]
        self.lam[k + 1] = res["lam_new"]
        self.gam[k] = res["gamma_k_new"]
        self.gam[k + 1] = res["gamma_k1_new"]
        plan.destroy()
        return res["discarded"]

    def apply_layer(self, parity: int, thetas, phis, chi_max: int, cutoff: float = 1e-14, contraction=None):
        """Gates on (k, k+1) for k = parity, parity+2, … < M−1; returns their discarded weights."""
        return [self.apply_gate(k, thetas[g], phis[g], chi_max, cutoff, contraction)
                for g, k in enumerate(range(parity, self.M - 1, 2))]
