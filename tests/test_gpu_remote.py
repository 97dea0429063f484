"""The SECTOR_OWNER exchange fused into K5 (tn_theta_exec_remote + CUDA IPC): two processes share the one
GPU, each computes its row shard and writes its slab of every Θ(c) straight into the owning process's
buffer; every owner then holds the full sectors it owns, bit-identical to the unsharded Θ. The ranks'
kernels never wait on each other (the only synchronisation is a host barrier after each stream drains),
so one GPU stands in for the NVLink peers without changing what the kernels do."""
import os
import socket

import numpy as np
import torch
import pytest
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


def _worker_pair(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import paper_2301_12814_b200 as tn
        import synth
        torch.cuda.set_device(0)
        c = synth.make_pair_config(cfg)
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        args = [dv(x) for x in (c.gamma_k, c.lam_k, c.gamma_k1, c.lam_l, c.lam_r)]
        full_plan = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
        full = [x.clone() for x in tn.theta_exec(full_plan, *args, tn.build_bs_unitary(full_plan, c.theta, c.phi))]
        plan = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r, world, rank)
        owned = tn.theta_exec_to_owners(plan, *args, tn.build_bs_unitary(plan, c.theta, c.phi))
        ok = all(torch.equal(v, full[s_]) for s_, v in owned.items())
        counts = [None] * world
        dist.all_gather_object(counts, len(owned))
        q.put((rank, "ok" if ok else "mismatch", sum(counts)))
    except Exception as e:
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, cfg, engine, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import paper_2301_12814_b200 as tn
        import synth
        from gpu_util import gpu_theta, to_dev
        torch.cuda.set_device(0)
        case = synth.make_config(cfg)
        _, _, full = gpu_theta(case, contraction=engine)          # unsharded reference, same GPU path
        plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, rank)
        if engine:
            plan.set_contraction(*engine)
        U = tn.build_bs_unitary(plan, case.theta, case.phi)
        t = to_dev(case)
        owned = tn.theta_exec_to_owners(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)
        ok = all(np.array_equal(v.cpu().numpy(), full[c]) for c, v in owned.items())
        counts = [None] * world
        dist.all_gather_object(counts, len(owned))
        q.put((rank, "ok" if ok else "mismatch", sum(counts)))
    except Exception as e:
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,engine", [(1, None), (2, None), (2, ("int8", 6))])
def test_exec_to_owners_two_processes_one_gpu(cfg, engine, cuda_ok):
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, engine, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] == "ok" for r in res), res
    c = synth.CONFIGS[cfg]
    assert res[0][2] >= 1


@pytest.mark.parametrize("cfg", [1, 2])
def test_exec_to_owners_pair_two_processes_one_gpu(cfg, cuda_ok):
    # MPO pair plans: each of two processes writes its row slabs of every Θ(c1,c2) into the owner's buffer
    # through CUDA IPC; the owners' sectors equal the unsharded pair exec bit for bit
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_pair, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] == "ok" for r in res), res
    c = synth.make_pair_config(cfg)
    full = tn_full_sector_count(c)
    assert res[0][2] == full


def tn_full_sector_count(c):
    import paper_2301_12814_b200 as tn
    p = tn.Plan2(c.d, c.N, c.q1_l, c.q2_l, c.q1_c, c.q2_c, c.q1_r, c.q2_r)
    return sum(1 for s in range(p.nsec) if p.sector_shape(s)[0] * p.sector_shape(s)[1] > 0)


def test_exec_remote_single_rank_and_errors(cuda_ok):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C
    import paper_2301_12814_b200 as tn
    import synth
    from gpu_util import gpu_theta, to_dev
    case = synth.make_config(1)
    _, _, full = gpu_theta(case)
    plan = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r)
    U = tn.build_bs_unitary(plan, case.theta, case.phi)
    t = to_dev(case)
    owned = tn.theta_exec_to_owners(plan, t["gk"], t["lk"], t["gk1"], t["ll"], t["lr"], U)   # world 1: all local
    assert set(owned) == {c for c in range(case.N + 1) if full[c].size}
    for c, v in owned.items():
        assert np.array_equal(v.cpu().numpy(), full[c])
    nulls = (C.c_void_p * plan.nsec)()
    with pytest.raises(tn.TnError, match="DIMENSION"):
        tn.check(tn.lib.tn_theta_exec_remote(plan.handle, None, *(tn._ptr(t[k]) for k in ("gk", "lk", "gk1", "ll", "lr")),
                                             tn._ptr(U), nulls), "tn_theta_exec_remote")
    # MPO pair plans: K5P's first pass runs in place on the local workspace, the second writes the owners' Θ
    pc = synth.make_pair_config(1)
    p2 = tn.Plan2(pc.d, pc.N, pc.q1_l, pc.q2_l, pc.q1_c, pc.q2_c, pc.q1_r, pc.q2_r)
    U2 = tn.build_bs_unitary(p2, pc.theta, pc.phi)
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    args2 = [dv(x) for x in (pc.gamma_k, pc.lam_k, pc.gamma_k1, pc.lam_l, pc.lam_r)]
    ref2 = [x.clone() for x in tn.theta_exec(p2, *args2, U2)]
    owned2 = tn.theta_exec_to_owners(p2, *args2, U2)
    assert set(owned2) == {s_ for s_ in range(p2.nsec) if ref2[s_].numel()}
    for s_, v in owned2.items():
        assert torch.equal(v, ref2[s_]), s_
    lit = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r).set_contraction("literal")
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        tn.check(tn.lib.tn_theta_exec_remote(lit.handle, None, *(tn._ptr(t[k]) for k in ("gk", "lk", "gk1", "ll", "lr")),
                                             tn._ptr(U), nulls), "tn_theta_exec_remote")
