"""Layer parallelism of the brick-wall TEBD (paper_2301_12814_b200.mps; PAPER.md:99
"beam splitter updates within a layer are parallel") — host logic on CPU with `gloo`, world 2 and 3.

Every rank holds a replica of the MPS; MPS.apply_layer(group=…) deals the gates by longest-processing-
time (layer_owners), runs its own and broadcasts the updated q, λ, Γ^{[k]}, Γ^{[k+1]}. The GPU gate is
replaced by the CPU oracle's gate (oracle/layer.py) in a test-only subclass that overrides apply_gate, so
the distributed run must reproduce the serial oracle layer bit for bit on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_gate(mps, k, theta, phi, chi_max, cutoff):
    import oracle.layer as L
    st = dict(N=mps.N, d=mps.d, q=[x.numpy() for x in mps.q], gam=[x.numpy() for x in mps.gam],
              lam=[x.numpy() for x in mps.lam], form="b")
    disc = L.apply_gate(st, k, theta, phi, chi_max, cutoff)
    for b in (k + 1,):
        mps.q[b] = torch.from_numpy(np.ascontiguousarray(st["q"][b]).astype(np.int32))
        mps.lam[b] = torch.from_numpy(np.ascontiguousarray(st["lam"][b]))
    for s in (k, k + 1):
        mps.gam[s] = torch.from_numpy(np.ascontiguousarray(st["gam"][s]))
    return disc


def _oracle_gate2(mpo, k, theta, phi, chi_max, cutoff):
    import oracle.layer as L
    st = dict(N=mpo.N, d=mpo.d, q1=[x.numpy() for x in mpo.q1], q2=[x.numpy() for x in mpo.q2],
              gam=[x.numpy() for x in mpo.gam], lam=[x.numpy() for x in mpo.lam], form="b")
    disc = L.apply_gate2(st, k, theta, phi, chi_max, cutoff)
    mpo.q1[k + 1] = torch.from_numpy(np.ascontiguousarray(st["q1"][k + 1]).astype(np.int32))
    mpo.q2[k + 1] = torch.from_numpy(np.ascontiguousarray(st["q2"][k + 1]).astype(np.int32))
    mpo.lam[k + 1] = torch.from_numpy(np.ascontiguousarray(st["lam"][k + 1]))
    for s in (k, k + 1):
        mpo.gam[s] = torch.from_numpy(np.ascontiguousarray(st["gam"][s]))
    return disc


def _worker_mpo(rank, world, port, M, N, d, chi, chi_max, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle.layer as L
        from paper_2301_12814_b200.mps import MPO
        st = L.random_mpo(M, N, d, chi, seed)
        ref = L.copy_state2(L.to_bform(st))   # the MPO class keeps right-canonical tensors
        class OracleMPO(MPO):  # test subclass: the GPU gate replaced by the oracle's
            def apply_gate(self, k, theta, phi, chi_max, cutoff=1e-14, contraction=None):
                return _oracle_gate2(self, k, theta, phi, chi_max, cutoff)

        mpo = OracleMPO.from_state(st, device="cpu")
        rng = np.random.default_rng(seed + 9)
        for parity in (0, 1, 0):
            n = len(range(parity, M - 1, 2))
            th, ph = rng.uniform(0, np.pi / 2, n), rng.uniform(0, 2 * np.pi, n)
            d_ref = L.apply_layer2(ref, parity, th, ph, chi_max)
            d_par = mpo.apply_layer(parity, th, ph, chi_max, group=dist.group.WORLD)
            assert d_par == [float(x) for x in d_ref], (rank, parity)
            got = mpo.to_state()
            for b in range(M + 1):
                assert np.array_equal(got["q1"][b], ref["q1"][b]) and np.array_equal(got["q2"][b], ref["q2"][b])
                assert np.array_equal(got["lam"][b], ref["lam"][b]), (rank, parity, b)
            for s_ in range(M):
                assert np.array_equal(got["gam"][s_], ref["gam"][s_]), (rank, parity, s_)
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, M, N, d, chi, chi_max, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle.layer as L
        from paper_2301_12814_b200.mps import MPS
        st = L.random_mps(M, N, d, chi, seed)
        ref = L.copy_state(L.to_bform(st))    # the MPS class keeps right-canonical tensors
        class OracleMPS(MPS):  # test subclass: the GPU gate replaced by the oracle's
            def apply_gate(self, k, theta, phi, chi_max, cutoff=1e-14, contraction=None):
                return _oracle_gate(self, k, theta, phi, chi_max, cutoff)

        mps = OracleMPS.from_state(st, device="cpu")
        rng = np.random.default_rng(seed + 7)
        for parity in (0, 1, 0, 1):
            n = len(range(parity, M - 1, 2))
            th, ph = rng.uniform(0, np.pi / 2, n), rng.uniform(0, 2 * np.pi, n)
            d_ref = L.apply_layer(ref, parity, th, ph, chi_max)
            d_par = mps.apply_layer(parity, th, ph, chi_max, group=dist.group.WORLD)
            assert d_par == [float(x) for x in d_ref], (rank, parity)
            got = mps.to_state()
            for b in range(M + 1):
                assert np.array_equal(got["q"][b], ref["q"][b]), (rank, parity, b)
                assert np.array_equal(got["lam"][b], ref["lam"][b]), (rank, parity, b)
            for s in range(M):
                assert np.array_equal(got["gam"][s], ref["gam"][s]), (rank, parity, s)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 7), (3, 8)])
def test_layer_parallel_matches_serial(world, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, 3, 4, 12, 9, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_mpo_layer_parallel_matches_serial():
    # the same exchange for MPO layers (two charge species per bond, U⊗U* gates): oracle apply_gate2 injected
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mpo, args=(r, world, port, 5, 2, 3, 6, 8, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_layer_owners_lpt():
    from paper_2301_12814_b200.mps import layer_owners
    assert layer_owners([5.0, 5.0, 5.0], 1) == [0, 0, 0]
    # decreasing cost, each to the least-loaded rank (ties → lower rank): 9→0, 7→1, 4→1, 3→0, 1→1
    assert layer_owners([3.0, 9.0, 4.0, 7.0, 1.0], 2) == [0, 0, 1, 1, 1]
    own = layer_owners([float(x) for x in range(1, 12)], 4)
    loads = [sum(c for c, o in zip(range(1, 12), own) if o == r) for r in range(4)]
    assert max(loads) - min(loads) <= 11 and sorted(set(own)) == [0, 1, 2, 3]
    assert layer_owners([], 3) == []
