"""A/B frame timing of the k = 6 near-kernel path on block1.67M (GPU box).

Each variant (environment switches, e.g. MGPBD_GJ_BIG_N=100000 or MGPBD_TILE_LONG_ROWS=1) runs in its own process:
frame 0 builds the hierarchy (no re-setups after it), then 3 more frames of 2 outer iterations each; prints the
per-frame device times and the level sizes.

  python tools/ab_frames_k6.py "" "MGPBD_TILE_LONG_ROWS=1"
"""
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
