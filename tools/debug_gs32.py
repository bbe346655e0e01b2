import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2505_13390_b200 import mgpbd, scenes
def rel(a,b): return np.linalg.norm(a-b)/np.linalg.norm(b)
for name in ("block_small","bar3k","cloth64"):
    sc = scenes.make(name) if name!="cloth64" else scenes.cloth(64, dt=3e-3, n_iters=5)
    for sm in (0,2):
        res={}
        for prec in (0,1):
            ctx=mgpbd.Context.from_scene(sc, smoother=sm, level0_operator=0, precision=prec)
            for it in (1,2,3,sc.n_iters):
                pass
            ctx.step(sc.dt, sc.n_iters); res[prec]=(ctx.lambdas(), ctx.stats().indefinite_events); ctx.close()
        print(name, "smoother", sm, "fp32 vs fp64 lambda rel %.2e" % rel(res[1][0], res[0][0]), "indef", res[0][1], res[1][1])
