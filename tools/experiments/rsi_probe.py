"""Numerics probe for an own-kernel phase A of the SVD step (DESIGN.md §7 Next (1)): randomized subspace
iteration on each config-3 sector Θ(c) with block b = k' + p and q power steps, Rayleigh–Ritz by the Gram of
Y = Θ·X, then the Ritz values against the exact singular values (torch.linalg.svdvals). Prototype in torch
(cuSOLVER QR / eigh) — it only measures whether the subspace is good enough. One GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

case = synth.make_config(3)
h = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
U = tn.build_bs_unitary(plan, case.theta, case.phi)
out = tn.theta_exec(plan, h(case.gamma_k), h(case.lam_k), h(case.gamma_k1), h(case.lam_l), h(case.lam_r), U)
torch.cuda.synchronize()
svals = [torch.linalg.svdvals(o) if o.numel() else torch.zeros(0, dtype=torch.float64, device="cuda") for o in out]
allv = torch.cat(svals)
T = torch.sort(allv, descending=True).values[4095].item()
s1 = allv.max().item()
g = torch.Generator(device="cuda").manual_seed(0)
for c, o in enumerate(out):
    if o.numel() == 0:
        continue
    A = o if o.shape[0] >= o.shape[1] else o.conj().T
    m, n = A.shape
    kp = int((svals[c] >= T).sum().item())
    if n < 600 or kp == 0:
        continue
    ex = svals[c][:kp]
    for p in (64, 128, 256):
        for q in (1, 2, 3):
            b = min(n, kp + p)
            om = torch.complex(torch.randn(n, b, generator=g, device="cuda", dtype=torch.float64),
                               torch.randn(n, b, generator=g, device="cuda", dtype=torch.float64))
            Q, _ = torch.linalg.qr(A @ om)
            for _ in range(q):
                X, _ = torch.linalg.qr(A.conj().T @ Q)
                Q, _ = torch.linalg.qr(A @ X)
            X, _ = torch.linalg.qr(A.conj().T @ Q)
            Y = A @ X
            w, V = torch.linalg.eigh(Y.conj().T @ Y)
            Y2 = Y @ V
            nrm = torch.linalg.vector_norm(Y2, dim=0)
            M = Y2.conj().T @ Y2
            d = torch.sqrt(torch.diagonal(M).real)
            rho = (M.abs() / (d[:, None] * d[None, :])).fill_diagonal_(0).max().item()
            rv = torch.sort(nrm, descending=True).values[:kp]
            err = (rv - ex).abs().max().item() / s1
            print(json.dumps({"sector": c, "m": m, "n": n, "k'": kp, "p": p, "q": q, "b": b, "err_rel_s1": err,
                              "rho_after_RR": rho, "edge_ratio": (svals[c][min(n - 1, b)] / svals[c][kp - 1]).item()}),
                  flush=True)
