import sys; sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make("block1.67M")
ctx = mgpbd.Context.from_scene(sc, precision=1, k_nullspace=6, max_dense_coarse=8192, setup_interval=1000,
                               resetup_on_indef=0, profile=1)
for f in range(2):
    ctx.step(sc.dt, 1)
    st = ctx.stats(); print("frame", f, st.ms_frame, st.kernel_launches, flush=True)
