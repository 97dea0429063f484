"""Probe: cost of the SVD-step building blocks on one B200 for a config-3-sized sector (complex128).

Times (CUDA events, after a warm-up) torch's cuSOLVER/cuBLAS wrappers on an R×C matrix with a decaying
spectrum: full SVD drivers, values only, the Gram matrix X^H X (cuBLAS), the Hermitian eigensolver on it
(values only / with vectors), and the tall-skinny Rayleigh–Ritz step X·V_k → SVD. Decides whether a
Gram-eigen + Rayleigh–Ritz SVD step can beat Xgesvdp by enough to be worth building."""
import json
import sys

import torch


def tm(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 2)


R, C = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (2176, 2048)))
k = int(sys.argv[3]) if len(sys.argv) > 3 else 256
g = torch.Generator(device="cuda").manual_seed(1)
dev = "cuda"
m = min(R, C)
Q1, _ = torch.linalg.qr(torch.randn(R, m, dtype=torch.complex128, device=dev, generator=g))
Q2, _ = torch.linalg.qr(torch.randn(C, m, dtype=torch.complex128, device=dev, generator=g))
s = torch.logspace(0, -8, m, dtype=torch.float64, device=dev)
X = (Q1 * s) @ Q2.mH
out = {"R": R, "C": C, "k": k}
for drv in ("gesvd", "gesvdj", "gesvda"):
    try:
        out[f"svd_{drv}_ms"] = tm(lambda: torch.linalg.svd(X, full_matrices=False, driver=drv))
    except Exception as e:  # noqa: BLE001
        out[f"svd_{drv}_ms"] = str(e)[:80]
out["svdvals_ms"] = tm(lambda: torch.linalg.svdvals(X))
G = X.mH @ X
out["gram_ms"] = tm(lambda: X.mH @ X)
out["eigvalsh_ms"] = tm(lambda: torch.linalg.eigvalsh(G))
out["eigh_ms"] = tm(lambda: torch.linalg.eigh(G))
w, V = torch.linalg.eigh(G)
Vk = V[:, -k:]
out["rr_gemm_ms"] = tm(lambda: X @ Vk)
Y = X @ Vk
out["rr_svd_tall_ms"] = tm(lambda: torch.linalg.svd(Y, full_matrices=False))
out["rr_qr_ms"] = tm(lambda: torch.linalg.qr(Y))
Qy, Ry = torch.linalg.qr(Y)
out["rr_small_svd_ms"] = tm(lambda: torch.linalg.svd(Ry, full_matrices=False))
sy = torch.linalg.svdvals(Ry)
out["rr_top_k_rel_err"] = float(((sy - s[:k]).abs() / s[:k]).max())
out["gram_top_k_rel_err"] = float(((w.flip(0)[:k].clamp(min=0).sqrt() - s[:k]).abs() / s[:k]).max())
print(json.dumps(out), flush=True)
