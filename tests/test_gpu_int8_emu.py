"""GPU parity of the tcgen05 INT8 emulated-FP64 contraction (TN_CONTRACT_INT8_OZAKI) against the CPU oracle:
the same bar as the FP64 DMMA path — ≤ 1e-10 relative Frobenius per sector (BASELINE.json north_star),
oracle-zero sectors exactly zero, identical shapes."""
import functools

import numpy as np
import pytest

import synth
from gpu_util import assert_sectors_close, gpu_theta, oracle_theta, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def tn(cuda_ok):
    import paper_2301_12814_b200 as tn
    return tn


@functools.lru_cache(maxsize=None)
def _case(cfg, shuffled=False, flat=False):
    return synth.make_config(cfg, shuffled=shuffled, flat=flat)


@functools.lru_cache(maxsize=None)
def _oracle(cfg, shuffled=False, flat=False):
    return oracle_theta(_case(cfg, shuffled, flat))


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("variant", ["plain", "flat"])
def test_int8_emulation_parity(tn, cfg, variant):
    kw = dict(flat=variant == "flat")
    case = _case(cfg, **kw)
    ref, *_ = _oracle(cfg, **kw)
    plan, _, got = gpu_theta(case, contraction=("int8", 7))
    assert plan.contraction() == ("int8", 7)
    worst = assert_sectors_close(got, ref, TOL, f"int8 config{cfg}-{variant}")
    assert worst < 1e-11


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("variant", ["plain", "flat"])
def test_int8_emulation_parity_s6(tn, cfg, variant):
    # the slice count bench.py's alt_engine line uses (S = 6, R20): the same ≤ 1e-10 bar
    kw = dict(flat=variant == "flat")
    case = _case(cfg, **kw)
    ref, *_ = _oracle(cfg, **kw)
    plan, _, got = gpu_theta(case, contraction=("int8", 6))
    assert plan.contraction() == ("int8", 6)
    assert_sectors_close(got, ref, TOL, f"int8 S=6 config{cfg}-{variant}")


@pytest.mark.parametrize("slices", [5, 8])
def test_int8_emulation_slices(tn, slices):
    # S = 8 meets the bar with margin; S = 5 is the documented failure (≈ 1e-9, R20) — it must be
    # worse than 1e-10 somewhere yet still close (a wrong slice layout would be O(1))
    case = _case(2)
    ref, *_ = _oracle(2)
    _, _, got = gpu_theta(case, contraction=("int8", slices))
    if slices >= 6:
        assert_sectors_close(got, ref, TOL, f"int8 S={slices}")
    else:
        worst = max(rel_err(g, r) for g, r in zip(got, ref))
        assert 1e-12 < worst < 1e-6, worst


def test_int8_vs_dmma_agree(tn):
    case = _case(2, shuffled=True)
    _, _, a = gpu_theta(case)
    _, _, b = gpu_theta(case, contraction=("int8", 7))
    for x, y in zip(a, b):
        assert rel_err(y, x) < 1e-11


@pytest.mark.parametrize("name,N,d,chi", [("N0", 0, 2, (3, 2, 4)), ("chi1", 3, 4, (1, 1, 1)),
                                          ("d_lt_N1", 6, 3, (40, 33, 29)), ("ragged", 5, 6, (131, 67, 190))])
def test_int8_edge_cases(tn, name, N, d, chi):
    case = synth.make_case(N, d, *chi, seed=17, charges="uniform", lam="random")
    ref, *_ = oracle_theta(case)
    _, _, got = gpu_theta(case, contraction=("int8", 7))
    assert_sectors_close(got, ref, 1e-10, name)


def test_int8_sharded_equals_unsharded(tn):
    case = _case(2)
    _, _, full = gpu_theta(case, contraction=("int8", 7))
    world = 4
    slabs = [[] for _ in range(case.N + 1)]
    for r in range(world):
        pr = tn.Plan(case.d, case.N, case.q_l, case.q_c, case.q_r, world, r)
        _, _, loc = gpu_theta(case, world, r, plan=pr, contraction=("int8", 7))
        for c in range(case.N + 1):
            slabs[c].append((pr.local_sector_shape(c)[2], loc[c]))
    for c in range(case.N + 1):
        parts = sorted((x for x in slabs[c] if x[1].shape[0] > 0), key=lambda x: x[0])
        if parts:
            assert np.array_equal(np.concatenate([p for _, p in parts], axis=0), full[c])


def test_set_contraction_errors(tn):
    plan = tn.Plan(4, 3, [0, 1], [0, 1], [0, 1])
    with pytest.raises(tn.TnError, match="DOMAIN"):
        plan.set_contraction("int8", 3)
    with pytest.raises(tn.TnError, match="DOMAIN"):
        plan.set_contraction(5, 7)
    plan.set_contraction("dmma")
    assert plan.contraction() == ("dmma", 0)
    # the int32 diagonal accumulators are exact only for K ≤ 2048 (OZ_KMAX): a longer centre segment is refused
    big = tn.Plan(4, 3, [1, 2, 3], np.zeros(2100, dtype=np.int32), [0, 1])
    with pytest.raises(tn.TnError, match="UNSUPPORTED"):
        big.set_contraction("int8", 6)
    assert big.contraction() == ("dmma", 0)      # the plan stays usable on the FP64 engine
