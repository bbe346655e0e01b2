"""Convergence / scaling experiments of SURVEY.md §8(f) row f3 on the synthetic scenes (GPU, C-ABI).

  python tools/experiments.py [linearity] [lazy] [smoother] [cloth_tol]

* linearity — time per outer iteration vs problem size (Fig. 8a: "linearly scaled up
  with resolution"): cloth N x N and block slabs of growing length; least-squares line and R^2.
* lazy — setup interval 1/10/20/50/100 (Fig. 5) on block_small over 100 frames: mean
  relative residual ||b_last|| / ||b_0|| per frame, frames with a setup, device time.
* smoother — omega-Jacobi vs Chebyshev ("omega-Jacobi has the best performance for
  softbody, and Chebyshev has the best performance for cloth") at the same number of matrix passes.
* omega_refresh — indefinite MGPCG steps through the lazy window (reading c26): bar50k and block1.67M
  frames in the literal lazy schedule (no early re-setup), omega_refresh_iters 0 / 10 / 50, lambda_safety 1 / 1.1:
  indefinite PCG iterations per frame, residual reduction, device time.
* cloth_tol — the paper's cloth hanging test (Fig. cloth, Table 1: N = 64/128/256/512, dt 3 ms,
  stiffness 1e9, "maxiter (1e5) ... ||b|| < 1e-4"): outer iterations and device time per frame until
  ||b|| < 1e-4 (absolute, Alg. 1 l.12), capped at MAXIT.
Prints one JSON object per experiment.
"""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402


def steady_ms_per_iter(sc, n_iters, frames=3, **kw):
    ctx = mgpbd.Context.from_scene(sc, precision=1, **kw)
    ms = []
    for f in range(frames):
        ctx.step(sc.dt, n_iters)
        st = ctx.stats()
        if not st.setup_ran:
            ms.append(st.ms_frame / n_iters)
    ctx.close()
    return min(ms)


def fit(xs, ys):
    xs, ys = np.asarray(xs, float), np.asarray(ys, float)
    a, b = np.polyfit(xs, ys, 1)
    r2 = 1 - ((ys - (a * xs + b)) ** 2).sum() / ((ys - ys.mean()) ** 2).sum()
    return a, b, r2


def linearity():
    out = {}
    rows = []
    for n in (128, 256, 512, 1024, 2048):
        sc = scenes.cloth(n, dt=3e-3, n_iters=20)
        rows.append((sc.n_cons, steady_ms_per_iter(sc, 20)))
    a, b, r2 = fit(*zip(*rows))
    out["cloth"] = {"points": rows, "ms_per_iter_per_Mcons": a * 1e6, "intercept_ms": b, "r2": r2}
    rows = []
    for cells in (17, 34, 68, 136):
        sc = scenes.kuhn_block(cells, 64, 32, 0.01, dt=3e-3, squash=0.7, twist_deg=45.0 * cells / 136.0,
                               n_iters=20, name=f"blockslab{cells}")
        rows.append((sc.n_cons, steady_ms_per_iter(sc, 20)))
    a, b, r2 = fit(*zip(*rows))
    out["block"] = {"points": rows, "ms_per_iter_per_Mcons": a * 1e6, "intercept_ms": b, "r2": r2}
    print(json.dumps({"experiment": "linearity", **out}), flush=True)


def lazy():
    sc = scenes.make("block_small")
    res = {}
    for k in (1, 10, 20, 50, 100):
        ctx = mgpbd.Context.from_scene(sc, precision=1, setup_interval=k)
        rel, setups, ms = [], 0, 0.0
        for f in range(100):
            ctx.step(sc.dt, sc.n_iters)
            st = ctx.stats()
            rel.append(st.b_norm[st.n_b - 1] / st.b_norm[0])
            setups += st.setup_ran
            ms += st.ms_frame
        ctx.close()
        res[str(k)] = {"mean_rel_residual": statistics.mean(rel), "max_rel_residual": max(rel),
                       "setups": setups, "ms_total": ms}
    print(json.dumps({"experiment": "lazy_setup_interval", "scene": sc.name, "frames": 100, **res}), flush=True)


def smoother():
    """Per-frame constraint-residual reduction ||b_last|| / ||b_0|| (Alg. 1, fp32, mean over 10 frames)
    and frame time with the omega-Jacobi and the Chebyshev smoother at the same number of matrix passes.
    (A random right-hand side is not a useful probe: the dual matrix of a planar cloth has a near-null
    space of dimension ~m/3 regularised only by alpha/dt^2, which dominates ||A^-1 b|| for random b.)"""
    res = {}
    for name in ("cloth64", "cloth256", "block_small", "bar3k"):
        sc = scenes.make(name) if name != "cloth64" else scenes.cloth(64, dt=3e-3, n_iters=20)
        for sm in (0, 1):
            ctx = mgpbd.Context.from_scene(sc, precision=1, smoother=sm)
            rel, ms = [], []
            for f in range(10):
                ctx.step(sc.dt, sc.n_iters)
                st = ctx.stats()
                rel.append(st.b_norm[st.n_b - 1] / st.b_norm[0])
                if not st.setup_ran:
                    ms.append(st.ms_frame)
            ctx.close()
            res[f"{name}/{'chebyshev' if sm else 'omega-jacobi'}"] = {
                "mean_rel_residual": statistics.mean(rel), "ms_frame": statistics.median(ms)}
    print(json.dumps({"experiment": "smoother", **res}), flush=True)


def cloth_tol(maxit=20000, frames=2):
    out = []
    for n in (64, 128, 256, 512):
        sc = scenes.cloth(n, dt=3e-3, n_iters=20)
        ctx = mgpbd.Context.from_scene(sc, precision=0, residual_abs=1e-4)
        rows = []
        for f in range(frames):
            ctx.step(sc.dt, maxit)
            st = ctx.stats()
            rows.append({"frame": f, "iters": st.iters_run, "b_first": st.b_norm[0], "b_last": st.b_last,
                         "ms": st.ms_frame, "converged": st.b_last < 1e-4})
        ctx.close()
        out.append({"N": n, "constraints": sc.n_cons, "frames": rows})
        print(json.dumps({"experiment": "cloth_tol", "N": n, "frames": rows}), flush=True)
    return out


def omega_refresh(frames=20):
    for name in ("bar50k", "block1.67M"):
        sc = scenes.make(name)
        for safety in (1.0, 1.1):
            for k in (0, 10, 50):
                ctx = mgpbd.Context.from_scene(sc, precision=1, lambda_safety=safety, resetup_on_indef=0,
                                               omega_refresh_iters=k)
                ev, rel, ms = [], [], []
                for f in range(frames):
                    ctx.step(sc.dt, sc.n_iters)
                    st = ctx.stats()
                    ev.append(st.indefinite_events)
                    rel.append(st.b_last / max(st.b_norm[0], 1e-300))
                    ms.append(st.ms_frame)
                ctx.close()
                print(json.dumps({"experiment": "omega_refresh", "config": name, "lambda_safety": safety,
                                  "omega_refresh_iters": k, "frames": frames, "indefinite_events": ev,
                                  "total_events": int(sum(ev)), "mean_rel_residual": statistics.mean(rel),
                                  "ms_frame_median": statistics.median(ms)}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["linearity", "lazy", "smoother"]
    for w in which:
        {"linearity": linearity, "lazy": lazy, "smoother": smoother, "cloth_tol": cloth_tol,
         "omega_refresh": omega_refresh}[w]()
