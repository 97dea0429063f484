"""Tiny Θ builds (BASELINE.json configs 0 and 1, both contraction engines) for compute-sanitizer runs
(SURVEY.md §8(c) T15): tools/gpu/sanitize.sh runs this under one sanitizer tool per gpurun call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import synth  # noqa: E402
from gpu_util import assert_sectors_close, gpu_theta, oracle_theta  # noqa: E402

for cfg in (0, 1):
    case = synth.make_config(cfg)
    ref, *_ = oracle_theta(case)
    for contraction in (None, ("int8", 7)):
        _, _, got = gpu_theta(case, contraction=contraction)
        w = assert_sectors_close(got, ref, 1e-10, f"config{cfg} {contraction}")
        print(f"config {cfg} contraction {contraction or 'dmma'}: worst sector rel err {w:.2e}", flush=True)
print("sanitize_case ok")
