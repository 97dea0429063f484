"""Host time of tn_theta_plan by phase (TN_PLAN_PROFILE=1 → stderr), config 3 at world 1 and every rank of
world 8, 30 plans each after warm-up; prints the median µs per phase. One GPU."""
import os
import re
import statistics
import subprocess
import sys

if os.environ.get("TN_PLAN_PROFILE") is None:
    env = dict(os.environ, TN_PLAN_PROFILE="1")
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    rows = {}
    for line in r.stderr.splitlines():
        m = re.match(r"\[plan\] world (\d+) rank (\d+) us: (.*) \(tiles", line)
        if not m:
            continue
        key = (int(m.group(1)), int(m.group(2)))
        vals = dict((k, float(v)) for k, v in re.findall(r"(\S+) ([\d.]+)", m.group(3)))
        rows.setdefault(key, []).append(vals)
    for key, v in sorted(rows.items()):
        v = v[5:]
        print(key, {k: round(statistics.median(x[k] for x in v), 1) for k in v[0]})
    print(r.stdout[-2000:])
    sys.exit(r.returncode)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12814_b200 as tn
import synth

case = synth.make_config(3)
hq = [np.ascontiguousarray(q) for q in (case.q_l, case.q_c, case.q_r)]
torch.cuda.init()
for world in (1, 8):
    for r in range(world):
        keep = []
        for i in range(35):
            keep.append(tn.Plan(case.d, case.N, *hq, world, r))
            if len(keep) > 3:
                keep.pop(0).destroy()
            torch.cuda.synchronize()
        for p in keep:
            p.destroy()
print("ok")
