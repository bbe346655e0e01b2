"""V-cycle / MGPCG of the full block with and without the cluster tail (same hierarchy inputs)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "block1.67M"
sc = scenes.make(name)
b = np.random.default_rng(7).normal(size=sc.n_cons)
for prec in (0, 1):
    out = {}
    for tail in (True, False):
        if tail:
            os.environ.pop("MGPBD_NO_TAIL", None)
        else:
            os.environ["MGPBD_NO_TAIL"] = "1"
        ctx = mgpbd.Context.from_scene(sc, precision=prec)
        ctx.debug_prepare(sc.dt)
        out[tail] = (ctx.debug_vcycle(b), ctx.debug_pcg(b, 5))
        ctx.close()
    rv = np.linalg.norm(out[True][0] - out[False][0]) / np.linalg.norm(out[False][0])
    rp = np.linalg.norm(out[True][1] - out[False][1]) / np.linalg.norm(out[False][1])
    print(f"{name} prec {prec}: tail vs no tail: V-cycle {rv:.3e}, 5-step PCG {rp:.3e}", flush=True)
