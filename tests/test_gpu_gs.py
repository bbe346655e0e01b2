"""GPU parity of the multicolour symmetric Gauss-Seidel smoother (
reading c22: forward colour order for pre-smoothing, reversed for post-smoothing) against the oracle,
through the C-ABI.  GS needs the assembled level-0 matrix (level0_operator = 0) and one rank."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu


def make_scene(name):
    if name == "cloth64":
        return scenes.cloth(64, dt=3e-3, n_iters=5)
    return scenes.make(name)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("sweeps", [1, 2])
@pytest.mark.parametrize("name", ["bar3k", "block_small"])
def test_gs_vcycle_pcg_identical_hierarchy(name, sweeps):
    sc = make_scene(name)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    h = O.Hierarchy(r, c, v, O.default_config(smoother=2, smoother_sweeps=sweeps))
    ctx = mgpbd.Context.from_scene(sc, smoother=2, smoother_sweeps=sweeps, level0_operator=0)
    ctx.debug_setup_from(v)
    b = np.random.default_rng(0).normal(size=sc.n_cons)
    assert rel(ctx.debug_vcycle(b), h.vcycle(b)) <= 1e-11
    for K in (1, 5):
        xo, rc, _ = h.pcg(b, K)
        assert rc == 0 and rel(ctx.debug_pcg(b, K), xo) <= 1e-9, K


# fp32 + GS on the squashed block: the GS update replaces x_i by a quotient of nearly cancelling
# fp32-stored terms, and the frame deviates 2.2e-3 from fp64 (the GPU's own fp64 GS frame matches the
# oracle to 1e-12; the case below pins the 5e-3 bound).  The omega-Jacobi default stays at ~1e-4.
CASES = [(n, 0, 1e-6) for n in ("cloth16", "cloth64", "bar3k", "block_small")] + \
        [(n, 1, 1e-3) for n in ("cloth16", "cloth64", "bar3k")] + [("block_small", 1, 5e-3)]


@pytest.mark.parametrize("name,precision,tol", CASES)
def test_gs_frame(name, precision, tol):
    sc = make_scene(name)
    ctx = mgpbd.Context.from_scene(sc, smoother=2, level0_operator=0, precision=precision)
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, smoother=2))
    ctx.step(sc.dt, sc.n_iters)
    sim.step(sc.dt, sc.n_iters)
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= tol and rel(ctx.positions() - sc.pos, xo - sc.pos) <= tol


def test_gs_config_errors():
    sc = scenes.make("cloth16")
    with pytest.raises(mgpbd.MgpbdError):
        mgpbd.Context.from_scene(sc, smoother=2)          # matrix-free level 0 cannot run GS
