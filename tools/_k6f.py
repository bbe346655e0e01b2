import sys, time; sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make("block1.67M")
ctx = mgpbd.Context.from_scene(sc, precision=1, k_nullspace=6, max_dense_coarse=8192)
for f in range(int(sys.argv[1]) if len(sys.argv) > 1 else 14):
    t = time.perf_counter()
    ctx.step(sc.dt, sc.n_iters)
    w = 1e3 * (time.perf_counter() - t)
    st = ctx.stats()
    print(f"frame {f} wall {w:.1f} event {st.ms_frame:.1f} setup {st.ms_setup:.1f} launches {st.kernel_launches} indef {st.indefinite_events} levels {[st.n[l] for l in range(st.n_levels)]}", flush=True)
