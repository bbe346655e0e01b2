"""Diagnose a GPU-vs-oracle frame mismatch: the same frame under every kernel-variant switch.

  python tools/diag_parity.py --config blockslab32 --iters 1 20 [--precision fp64]
"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

VARIANTS = [("default", {}), ("NO_TMA", {"MGPBD_NO_TMA": "1"}), ("NO_RES_COARSE", {"MGPBD_NO_RES_COARSE": "1"}),
            ("NO_COARSE_KERNEL", {"MGPBD_NO_COARSE_KERNEL": "1"}), ("NO_GRAPH", {"MGPBD_NO_GRAPH": "1"}),
            ("NO_GJ_COOP", {"MGPBD_NO_GJ_COOP": "1"}), ("NO_VA_SETUP", {"MGPBD_NO_VA_SETUP": "1"}),
            ("csr_level0", {"DIAG_OP": "0"})]


def child(cfg, iters, prec, out):
    import numpy as np
    from paper_2505_13390_b200 import mgpbd, scenes
    sc = scenes.make(cfg)
    op = int(os.environ.get("DIAG_OP", "1"))
    res = {}
    for n in iters:
        ctx = mgpbd.Context.from_scene(sc, precision=prec, level0_operator=op)
        ctx.step(sc.dt, n)
        res[n] = (ctx.lambdas(), ctx.positions())
        ctx.close()
    np.savez(out, **{f"l{n}": res[n][0] for n in iters}, **{f"x{n}": res[n][1] for n in iters})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="blockslab32")
    ap.add_argument("--iters", type=int, nargs="+", default=[1, 20])
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--child", default="")
    a = ap.parse_args()
    prec = 1 if a.precision == "fp32" else 0
    if a.child:
        return child(a.config, a.iters, prec, a.child)
    import numpy as np
    import oracle as O
    from paper_2505_13390_b200 import scenes
    sc = scenes.make(a.config)
    ref = {}
    for n in a.iters:
        sim = O.Sim(sc)
        sim.step(sc.dt, n)
        x, _, lam = sim.state()
        ref[n] = (lam, x)
    for name, env in VARIANTS:
        out = f"/tmp/diag_{name}.npz"
        r = subprocess.run([sys.executable, __file__, "--config", a.config, "--precision", a.precision, "--iters",
                            *map(str, a.iters), "--child", out], env={**os.environ, **env}, capture_output=True, text=True)
        if r.returncode != 0:
            print(name, "FAILED", r.stderr[-400:])
            continue
        d = np.load(out)
        msg = []
        for n in a.iters:
            lo, xo = ref[n]
            lg, xg = d[f"l{n}"], d[f"x{n}"]
            msg.append(f"n={n}: lambda {np.linalg.norm(lg - lo) / np.linalg.norm(lo):.2e} "
                       f"dx {np.linalg.norm((xg - sc.pos) - (xo - sc.pos)) / np.linalg.norm(xo - sc.pos):.2e}")
        print(f"{name:18s}", " | ".join(msg), flush=True)


if __name__ == "__main__":
    main()
