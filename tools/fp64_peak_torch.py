"""Library ceiling for the Θ contraction: cuBLAS DGEMM / ZGEMM through torch."""
import json
import torch

def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = (8 if dtype.is_complex else 2) * n ** 3
    return {"kind": f"torch_matmul_{str(dtype).split('.')[-1]}", "n": n, "ms": round(ms, 3),
            "tflops": round(fl / ms / 1e9, 2)}

for dt in (torch.float64, torch.complex128):
    for n in (2048, 4096, 8192):
        print(json.dumps(bench(dt, n)))
