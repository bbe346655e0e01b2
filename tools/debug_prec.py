import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make(sys.argv[1])
res = {}
for prec in (0, 1):
    ctx = mgpbd.Context.from_scene(sc, precision=prec, setup_interval=2)
    res[prec] = []
    for f in range(3):
        ctx.step(sc.dt, 4); res[prec].append((ctx.lambdas().copy(), ctx.positions().copy()))
for f in range(3):
    l0, l1 = res[0][f][0], res[1][f][0]
    x0, x1 = res[0][f][1] - sc.pos, res[1][f][1] - sc.pos
    print(f, "fp32 vs fp64 lam rel", np.linalg.norm(l1-l0)/np.linalg.norm(l0), "dx rel", np.linalg.norm(x1-x0)/np.linalg.norm(x0))
