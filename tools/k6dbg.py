import sys, os
sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
for name in sys.argv[1:]:
    sc = scenes.make(name)
    for prec in (0, 1):
        ctx = mgpbd.Context.from_scene(sc, precision=prec, k_nullspace=6)
        try:
            ctx.step(sc.dt, 2)
            st = ctx.stats()
            print(name, prec, "ok", [st.n[l] for l in range(st.n_levels)], flush=True)
        except Exception as e:
            try:
                st = ctx.stats(); lv = [st.n[l] for l in range(st.n_levels)]
            except Exception:
                lv = None
            print(name, prec, "FAIL", e, lv, flush=True)
        ctx.close()
