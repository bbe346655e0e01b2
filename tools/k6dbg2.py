import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
name = sys.argv[1]
sc = scenes.make(name)
ctx = mgpbd.Context.from_scene(sc, precision=0, k_nullspace=6)
ctx.debug_prepare(sc.dt)
st = ctx.stats()
nl = st.n_levels
print("levels", [st.n[l] for l in range(nl)], "omega", [st.omega[l] for l in range(nl)], flush=True)
for l in range(1, nl):
    r, c, v = ctx.level(l)
    n = len(r) - 1
    d = v[r[1:] - 1]
    print(l, "n", n, "nnz", len(v), "finite", np.isfinite(v).all(), "min diag", d.min(), "max |v|", np.abs(v).max(),
          "diag<=0", int((d <= 0).sum()), flush=True)
for l in range(nl - 1):
    pr, pc, pv = ctx.prolongator_csr(l)
    print("P", l, "finite", np.isfinite(pv).all(), "max", np.abs(pv).max(), "rows w/o entries", int((np.diff(pr) == 0).sum()), flush=True)
b = np.random.default_rng(0).normal(size=sc.n_cons)
z = ctx.debug_vcycle(b)
print("vcycle finite", np.isfinite(z).all(), "b.z", float(b @ z), flush=True)
