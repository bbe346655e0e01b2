import os, subprocess, sys
CH = r'''
import sys; sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make("block1.67M")
ctx = mgpbd.Context.from_scene(sc, precision=1, k_nullspace=6, max_dense_coarse=8192, setup_interval=1000, resetup_on_indef=0)
ms = []
for f in range(4):
    ctx.step(sc.dt, 2)
    ms.append(ctx.stats().ms_frame)
st = ctx.stats()
print("frames", [round(v, 2) for v in ms], "levels", [(st.n[l], st.nnz[l]) for l in range(st.n_levels)], flush=True)
'''
for var in sys.argv[1:] or [""]:
    env = dict(os.environ)
    for kv in var.split():
        k, v = kv.split("="); env[k] = v
    r = subprocess.run([sys.executable, "-c", CH], env=env, capture_output=True, text=True, timeout=900)
    print(repr(var), r.stdout.strip() or r.stderr[-500:], flush=True)
