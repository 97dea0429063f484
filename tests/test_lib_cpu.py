"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/tn_theta.h declares,
and its host-only logic (flop-balanced row shards, status strings) behaves. No compute call here
needs a GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "tn_theta.h")).read()
    return sorted(set(re.findall(r"^TN_API\s+[\w\s\*]+?\b(tn_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    syms = _header_symbols()
    for s in ("tn_theta_plan", "tn_build_bs_unitary", "tn_theta_exec", "tn_theta_exec_sharded"):
        assert s in syms


def test_library_exports_every_header_symbol():
    import paper_2301_12814_b200 as tn
    out = subprocess.run(["nm", "-D", "--defined-only", tn.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tn_\w+)$", out, flags=re.M))
    missing = [s for s in _header_symbols() if s not in exported]
    assert not missing, missing
    from paper_2301_12814_b200._lib import SIGNATURES
    assert set(SIGNATURES) == set(_header_symbols())


def test_library_is_sm100a():
    import paper_2301_12814_b200 as tn
    out = subprocess.run(["cuobjdump", "--list-elf", tn.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version():
    from paper_2301_12814_b200._lib import lib, STATUS
    for k, v in STATUS.items():
        assert lib.tn_status_string(k).decode() == v
    assert lib.tn_version() >= 1


def _cost_rows(d, N, nl, nc, nr):
    """Independent re-statement of the per-row device-time model the shard split balances: the
    row's K4 contraction flops (SURVEY.md §8(d), 8 per complex MAC) plus 355 flop-equivalents per Θ element it
    owns (K5 moves 32 B per element at ~3.7 TB/s while K4 runs at ~41 TFLOP/s)."""
    C = [sum(nr[max(0, c - d + 1):c + 1]) for c in range(N + 1)]
    cost = np.zeros(N + 1)
    for cl in range(N + 1):
        f = 0.0
        for cc in range(max(0, cl - d + 1), cl + 1):
            if nc[cc]:
                f += 8.0 * nc[cc] * C[cc]
        el = sum(C[c] for c in range(max(0, cl - d + 1), cl + 1))
        cost[cl] = f + 355.0 * el
    return cost


@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_rows_host_balanced(cfg, world):
    import paper_2301_12814_b200 as tn
    import synth
    N, d, ql, qc, qr = synth.make_charges(cfg)
    nl, nc, nr = (np.bincount(q, minlength=N + 1) for q in (ql, qc, qr))
    b = tn.shard_rows_host(d, N, nl, nc, nr, world)
    assert b[0] == 0 and b[-1] == len(ql) and np.all(np.diff(b) >= 0)
    cost = _cost_rows(d, N, nl, nc, nr)
    row_cost = np.repeat(cost, nl)
    per = np.array([row_cost[b[r]:b[r + 1]].sum() for r in range(world)])
    assert per.max() / per.mean() < 1.02 + (0.0 if cfg > 1 else 0.05)


def test_shard_rows_host_errors():
    import paper_2301_12814_b200 as tn
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.shard_rows_host(1, 3, [1] * 4, [1] * 4, [1] * 4, 2)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        tn.shard_rows_host(4, 3, [1] * 4, [1] * 4, [1] * 4, 0)


def test_null_plan_is_rejected_without_touching_cuda():
    import paper_2301_12814_b200 as tn
    for name, args in (("tn_plan_reserve", (None, 2)), ("tn_plan_exec_launches", (None, None))):
        with pytest.raises(tn.TnError, match="NULL"):
            tn.check(getattr(tn.lib, name)(*args), name)
