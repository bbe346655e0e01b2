"""Small frames that exercise every kernel family (for compute-sanitizer memcheck / racecheck / synccheck):
cloth16 fp64 + fp32 (CSR and matrix-free), block_small with min_coarse = 30 (TMA row kernel, persistent
coarse kernels, cluster tail, cooperative coarsest inverse, graphs), bar_small k = 6 (f2 kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402

runs = [("cloth16", dict(precision=0)), ("cloth16", dict(precision=1, level0_operator=0)),
        ("block_small", dict(precision=1, min_coarse=30)), ("block_small", dict(precision=0, min_coarse=30)),
        ("bar3k", dict(precision=0, k_nullspace=6))]
for name, kw in runs:
    sc = scenes.make(name)
    ctx = mgpbd.Context.from_scene(sc, **kw)
    for _ in range(2):
        ctx.step(sc.dt, 3)
    st = ctx.stats()
    print(name, kw, "levels", st.n_levels, "launches", st.kernel_launches, flush=True)
    ctx.close()
