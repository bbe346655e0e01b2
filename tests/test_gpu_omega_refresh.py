"""GPU parity of the optional per-frame omega refresh (reading c26, cfg.omega_refresh_iters > 0).

With the lazy setup every 100 frames, frames 1..3 run no setup: at ite 0 both sides re-estimate
lambda_max(D^-1 A_l) of every smoothed level with `omega_refresh_iters` power iterations on the current
fp64 level matrices, started from the iterate the previous estimate left.  Each frame restarts from the
oracle's end-of-frame state (as in test_gpu_literal.py), so the refreshed omegas are compared at 1e-9 and
lambda / x / v element-wise; the omegas must move between frames (the refresh ran)."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

SCHED = dict(setup_interval=100, resetup_on_indef=0, omega_refresh_iters=12)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("precision", [0, 1], ids=["fp64", "fp32"])
@pytest.mark.parametrize("name,extra", [("bar3k", {}), ("cloth64", {}), ("block_small", {}),
                                        ("bar3k", {"level0_operator": 0}), ("bar3k", {"k_nullspace": 3}),
                                        ("bar3k", {"smoother": 1})],
                         ids=["bar3k", "cloth64", "block_small", "bar3k-csr", "bar3k-k3", "bar3k-cheb"])
def test_omega_refresh_frames(name, extra, precision):
    sc = scenes.make(name)
    okw = {k: v for k, v in extra.items() if k != "level0_operator"}
    cfg = O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, **SCHED, **okw)
    sim = O.Sim(sc, cfg)
    ctx = mgpbd.Context.from_scene(sc, precision=precision, **SCHED, **extra)
    tol = 1e-6 if precision == 0 else 1e-3
    x_start = sc.pos.copy()
    prev = None
    for f in range(4):
        ctx.step(sc.dt, sc.n_iters)
        assert sim.step(sc.dt, sc.n_iters) == 0
        st = ctx.stats()
        assert st.setup_ran == (1 if f == 0 else 0) and sim.setups() == 1
        h = sim.hierarchy()
        assert st.n_levels == h.n_levels
        om = [h.omega(l) for l in range(h.n_levels - 1)]
        for l, o in enumerate(om):
            assert abs(st.omega[l] - o) <= 1e-9 * o, (f, l, st.omega[l], o)
        if prev is not None:
            assert max(abs(a - b) / b for a, b in zip(om, prev)) > 1e-12  # the refresh moved omega
        prev = om
        xo, vo, lo = sim.state()
        xg, vg, lg = ctx.positions(), ctx.velocities(), ctx.lambdas()
        el, ex, ev = rel(lg, lo), rel(xg - x_start, xo - x_start), rel(vg, vo)
        print(f"{name} {extra} fp{'32' if precision else '64'} frame {f}: lambda {el:.2e} dx {ex:.2e} v {ev:.2e}")
        if sim.indefinite_events() == 0 or precision == 0:
            assert el <= tol and ex <= tol and ev <= tol, (f, el, ex, ev)
        ctx.set_state(xo, vo)
        x_start = xo.copy()
    ctx.close()
