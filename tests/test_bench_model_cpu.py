"""bench.py's comm_model (the exchange steps the multi-GPU projection leaves out): its byte counts
come from the library's own host schedules (tn_shard_rows_host, tn_gather_schedule_host) and must add up to the
slabs and Θ blocks those schedules move. CPU only."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402


@pytest.mark.parametrize("cfg,R", [(2, 2), (2, 4), (3, 8)])
def test_comm_model_bytes(cfg, R):
    import paper_2301_12814_b200 as tn
    case = synth.make_config(cfg)
    hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
    per = [0.5] * R
    m = bench.comm_model(tn, case, hq, R, per, 4.0)
    chi_l, chi_c = len(case.q_l), len(case.q_c)
    cnt = [np.bincount(q, minlength=case.N + 1).astype(np.int64) for q in hq]
    b = tn.shard_rows_host(case.d, case.N, *cnt, R)
    # rank 0 sends every other rank its Γk rows
    assert m["slab_scatter_mb_rank0_sent"] == round((chi_l - (b[1] - b[0])) * chi_c * 16 / 1e6, 1)
    # the owner gather moves at most every Θ element once, and nothing when a rank owns its own rows
    theta_bytes = 0
    for c in range(case.N + 1):
        R_c = np.sum(cnt[0][c:min(case.N, c + case.d - 1) + 1])
        C_c = np.sum(cnt[2][max(0, c - case.d + 1):c + 1])
        theta_bytes += int(R_c) * int(C_c) * 16
    assert 0 < m["gather_owner_mb_max_sent"] * 1e6 <= theta_bytes
    # time model: bytes / nominal NVLink rate, and the speedups are ordered serial ≤ overlapped ≤ compute-only
    assert m["t_slab_ms"][0] == pytest.approx(m["slab_scatter_mb_rank0_sent"] * 1e6 / 900e9 * 1e3, rel=2e-3, abs=1e-4)
    # the root gather pulls every other rank's slabs into rank 0: more than any owner
    # receives, at most all of Θ, and never faster than the owner gather
    assert m["gather_owner_mb_max_recv"] <= m["gather_root_mb_recv"] <= theta_bytes / 1e6 + 0.1
    assert m["projected_speedup_slabs_and_root_gather_serial"] <= m["projected_speedup_slabs_and_owner_gather_serial"]
    for name in ("slabs", "full_bcast", "slabs_and_owner_gather", "slabs_and_root_gather"):
        s, o = m[f"projected_speedup_{name}_serial"], m[f"projected_speedup_{name}_overlapped"]
        assert s <= o <= 4.0 / max(per) + 1e-9


def _lines(name):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", name)
    import json
    with open(path) as f:
        return [json.loads(x) for x in f if x.strip()]


def test_bench_line_carries_the_contract_keys():
    # the committed closing bench line (profiles/r02_bench_final.jsonl) has every key the bench contract asks for
    for d in _lines("r02_bench_final.jsonl"):
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                  "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                  "gpu_launches", "clocks"):
            assert k in d, k
        assert d["warmup"] >= 3 and d["n_gpus"] == 1 and d["dtype"] == "f64" and "workload" in d["config"]
        r = d["roofline"]
        assert r["bound"] in ("hbm", "tensor", "alu") and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
        assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"]) and d["cpu_baseline"]["kind"] == "oracle"
        e = d["e2e"]
        assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["h2d_bytes_per_step"] > 0
        assert d["gpu_launches"] > 0 and not (set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                                                               "sw_thermal_slowdown"})
        # value = useful flops of the step / its time
        f = d["config"]["f_contract"] + d["config"]["f_mix"]
        assert d["value"] == pytest.approx(f / (d["ms_per_step"] * 1e-3) / 1e9, rel=2e-3)


def test_reference_line_carries_the_contract_keys():
    for d in _lines("r02_bench_ref.jsonl"):
        assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
        assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
        assert d["e2e"]["value"] == d["value"]
