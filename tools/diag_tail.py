"""V-cycle / MGPCG of the full block with and without the cluster tail (same hierarchy inputs)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "block1.67M"
sc = scenes.make(name)
b = np.random.default_rng(7).normal(size=sc.n_cons)
resetup = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # frames stepped before (B-type hierarchy: 2)
VARIANTS = {"solo": {"MGPBD_SOLO": "1"}, "fused": {}, "split": {"MGPBD_NO_FUSED_TAIL": "1"},
            "none": {"MGPBD_NO_TAIL": "1"}}
state = None
if resetup:  # a later state (B-type hierarchy), identical for every variant: stepped once by an fp64 context
    os.environ["MGPBD_NO_TAIL"] = "1"
    c0 = mgpbd.Context.from_scene(sc, precision=0)
    for _ in range(resetup):
        c0.step(sc.dt, 1)
    state = (c0.positions(), c0.velocities())
    c0.close()
for prec in (0, 1):
    out = {}
    for name_v, env in VARIANTS.items():
        for k in ("MGPBD_NO_TAIL", "MGPBD_NO_FUSED_TAIL", "MGPBD_SOLO"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ctx = mgpbd.Context.from_scene(sc, precision=prec)
        if state is not None:
            ctx.set_state(*state)
        ctx.setup_hierarchy()
        ctx.debug_prepare(sc.dt)
        out[name_v] = (ctx.debug_vcycle(b), ctx.debug_pcg(b, 5))
        ctx.close()
    for v in ("solo", "fused", "split"):
        rv = np.linalg.norm(out[v][0] - out["none"][0]) / np.linalg.norm(out["none"][0])
        rp = np.linalg.norm(out[v][1] - out["none"][1]) / np.linalg.norm(out["none"][1])
        print(f"{name} prec {prec}: {v} tail vs no tail: V-cycle {rv:.3e}, 5-step PCG {rp:.3e}", flush=True)
