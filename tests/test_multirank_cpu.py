"""World-size-2 `gloo` tests (CPU) of the N>1 host logic: every rank derives the same flop-balanced row
shards from the C library's host routine (tn_shard_rows_host, the rule tn_theta_plan uses), the
shards tile the sorted left positions, each rank's slab of every Θ(c) is rows(c) ∩ [r0, r1)
(include/tn_theta.h, tn_plan_local_sector_shape), and gathering the slabs on rank 0 reassembles the
full Θ (oracle values stand in for each rank's kernel output)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2301_12814_b200 as tn
        import synth
        case = synth.make_config(cfg, shuffled=True)
        N, d = case.N, case.d
        counts = [np.bincount(x, minlength=N + 1) for x in (case.q_l, case.q_c, case.q_r)]
        bounds = tn.shard_rows_host(d, N, *counts, world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds.tolist())
        assert all(b == allb[0] for b in allb), "ranks disagree on the shard bounds"
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        secs, perms, offs, _ = oracle.theta_sectors(N, d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
        slabs = []
        for c in range(N + 1):
            (a0, a1), _ = oracle.sector_ranges(offs[0], offs[2], N, d, c)
            l0, l1 = min(max(a0, r0), r1), min(max(a1, r0), r1)
            slabs.append((l0 - a0, secs[c][l0 - a0:l1 - a0]))
        gathered = [None] * world
        dist.all_gather_object(gathered, slabs)
        if rank == 0:
            for c in range(N + 1):
                # an empty slab's begin is clamped past the sector (no rows): only non-empty slabs tile
                parts = sorted((g[c] for g in gathered if g[c][1].shape[0] > 0), key=lambda x: x[0])
                pos = 0
                for begin, blk in parts:
                    assert begin == pos, "slabs must tile the sector rows"
                    pos += blk.shape[0]
                assert pos == secs[c].shape[0]
                full = np.concatenate([b for _, b in parts], axis=0) if parts else secs[c]
                assert np.array_equal(full, secs[c])
        q.put((rank, "ok", bounds.tolist()))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [0, 1])
def test_gloo_world2_shard_and_gather(cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
    b = res[0][2]
    assert b[0] == 0 and b[-1] == synth_chi(cfg) and b[1] > 0


def synth_chi(cfg):
    import synth
    return synth.CONFIGS[cfg]["chi"]


def _owner_worker(rank, world, port, cfg, q):
    """TN_GATHER_SECTOR_OWNER host logic over gloo: every rank derives the same owners from the library's
    rule, each sector's slabs are point-to-point sent to its owner (the exchange pattern of
    tn_theta_exec_sharded), and every owner reassembles its full sectors."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle
        import paper_2301_12814_b200 as tn
        import synth
        case = synth.make_config(cfg)
        N, d = case.N, case.d
        counts = [np.bincount(x, minlength=N + 1) for x in (case.q_l, case.q_c, case.q_r)]
        bounds = tn.shard_rows_host(d, N, *counts, world)
        secs, perms, offs, _ = oracle.theta_sectors(N, d, case.q_l, case.q_c, case.q_r, case.gamma_k, case.lam_k,
                                                    case.gamma_k1, case.lam_l, case.lam_r, case.theta, case.phi)
        sizes = [s.size for s in secs]
        owners = tn.sector_owners_host(sizes, world)
        allo = [None] * world
        dist.all_gather_object(allo, owners.tolist())
        assert all(o == allo[0] for o in allo)
        # LPT balance: no owner holds more than the mean plus the largest sector
        load = np.bincount(owners, weights=sizes, minlength=world)
        assert load.max() <= sum(sizes) / world + max(sizes)
        for c in range(N + 1):
            (a0, a1), _ = oracle.sector_ranges(offs[0], offs[2], N, d, c)
            o = int(owners[c])
            full = np.zeros_like(secs[c]) if rank == o else None
            for src in range(world):
                s0, s1 = min(max(a0, bounds[src]), a1), min(max(a0, bounds[src + 1]), a1)
                if s1 <= s0:
                    continue
                if src == rank and rank == o:
                    full[s0 - a0:s1 - a0] = secs[c][s0 - a0:s1 - a0]
                elif src == rank:
                    dist.send(torch.from_numpy(np.ascontiguousarray(secs[c][s0 - a0:s1 - a0])), dst=o)
                elif rank == o:
                    buf = torch.empty((s1 - s0, secs[c].shape[1]), dtype=torch.complex128)
                    dist.recv(buf, src=src)
                    full[s0 - a0:s1 - a0] = buf.numpy()
            if rank == o:
                assert np.array_equal(full, secs[c])
        q.put((rank, "ok", None))
    except Exception as e:
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [1])
def test_gloo_world2_sector_owner_gather(cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_owner_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_sector_owner_rule_is_lpt():
    import sys
    sys.path.insert(0, ROOT)
    import paper_2301_12814_b200 as tn
    sizes = [50, 10, 40, 30, 20, 0]
    # sorted 50,40,30,20,10,0 → r0, r1, r1 (40<50), r0 (50<70), r0 (tie 70=70 → lower), r1
    assert tn.sector_owners_host(sizes, 2).tolist() == [0, 0, 1, 1, 0, 1]
    assert tn.sector_owners_host(sizes, 1).tolist() == [0] * 6
