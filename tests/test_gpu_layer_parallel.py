"""Layer parallelism on the GPU ("beam splitter updates within a layer are
parallel"): two processes share the one GPU, each holding a replica of the MPS / MPO, and MPS.apply_layer(group=…)
deals the layer's gates to them (layer_owners), runs each rank's gates through the C ABI (Θ + SVD step on the GPU)
and broadcasts the updated tensors (gloo here, NCCL on a multi-GPU box). Every rank's replica must end each layer
bit-identical to the same layers run serially on the GPU, and within the layer-parity bar of the oracle. The ranks'
kernels never wait on each other (the exchange is host-mediated), so one GPU stands in for two without changing
what the kernels do."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle.layer as L
        from paper_2301_12814_b200.mps import MPO, MPS
        torch.cuda.set_device(0)
        if kind == "mps":
            st = L.random_mps(7, 3, 4, 12, 5)
            make = lambda: MPS.from_state(st)
            ref = L.to_bform(st)
            step = L.apply_layer
        else:
            st = L.random_mpo(5, 2, 3, 6, 3)
            nrm = np.linalg.norm(L.dense_state2(st)) ** (1.0 / 5)
            st["gam"] = [g / nrm for g in st["gam"]]
            make = lambda: MPO.from_state(st)
            ref = L.to_bform(st)
            step = L.apply_layer2
        par, ser = make(), make()
        rng = np.random.default_rng(77)
        for parity in (0, 1, 0, 1):
            n = len(range(parity, par.M - 1, 2))
            th, ph = rng.uniform(0, np.pi / 2, n), rng.uniform(0, 2 * np.pi, n)
            d_par = par.apply_layer(parity, th, ph, 9, group=dist.group.WORLD)
            d_ser = ser.apply_layer(parity, th, ph, 9)
            d_ref = step(ref, parity, th, ph, 9)
            assert d_par == [float(x) for x in d_ser], (rank, parity)
            a, b = par.to_state(), ser.to_state()
            for key in [k for k in ("q", "q1", "q2") if k in a]:
                for x, y in zip(a[key], b[key]):
                    assert np.array_equal(x, y), (rank, parity, key)
            for x, y in zip(a["lam"], b["lam"]):
                assert np.array_equal(x, y), (rank, parity, "lam")
            for x, y in zip(a["gam"], b["gam"]):
                assert np.array_equal(x, y), (rank, parity, "gam")
            for x, y in zip(a["lam"], ref["lam"]):
                assert np.max(np.abs(x - y), initial=0.0) <= 1e-10 * max(y.max(), 1e-300), (rank, parity)
        dense = L.dense_state if kind == "mps" else L.dense_state2
        got, want = dense(par.to_state()), dense(ref)
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["mps", "mpo"])
def test_layer_parallel_two_processes_match_serial(cuda_ok, kind):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"
