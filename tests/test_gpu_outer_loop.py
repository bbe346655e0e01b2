"""GPU parity of the Algorithm-1 outer-loop variants (reading c21): the
backtracking relaxation that halves omega when ||b|| rises and the ||b|| < eps exit of
Alg. 1 l.12, against the oracle through the C-ABI."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


# fp32 only on the cloth: on the 1e9-stiff bars the halving decision compares residual norms that
# differ by less than the fp32 rounding of the solve, so fp32 and fp64 can take different branches
@pytest.mark.parametrize("name,omega,precision", [("bar_small", 0.9, 0), ("bar3k", 0.9, 0), ("cloth64", 1.0, 0),
                                                  ("cloth64", 1.0, 1)])
def test_backtracking_frame(name, omega, precision):
    sc = scenes.make(name) if name != "cloth64" else scenes.cloth(64, dt=3e-3, n_iters=5)
    n_iters = 12
    ctx = mgpbd.Context.from_scene(sc, precision=precision, omega_relax=omega, backtrack=1)
    sim = O.Sim(sc, O.default_config(omega_relax=omega, pcg_iters=sc.pcg_iters, backtrack=1))
    ctx.step(sc.dt, n_iters)
    sim.step(sc.dt, n_iters)
    st = ctx.stats()
    xo, _, lo = sim.state()
    tol = 1e-6 if precision == 0 else 1e-3
    assert rel(ctx.lambdas(), lo) <= tol and rel(ctx.positions() - sc.pos, xo - sc.pos) <= tol
    if precision == 0:   # the halving decisions are taken on the same residual sequence
        assert st.omega_relax == sim.omega()
        assert np.allclose(np.array(st.b_norm[:n_iters]), sim.b_norms(n_iters), rtol=1e-6)


@pytest.mark.parametrize("name", ["bar3k", "block_small"])
def test_residual_exit_frame(name):
    sc = scenes.make(name)
    probe = O.Sim(sc)
    probe.step(sc.dt, 10)
    nb = probe.b_norms(10)
    tol = 1.001 * nb[:5].min() / nb[0]                 # the exit fires within the first 5 iterations
    ctx = mgpbd.Context.from_scene(sc, residual_tol=tol)
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, residual_tol=tol))
    ctx.step(sc.dt, 10)
    sim.step(sc.dt, 10)
    assert ctx.stats().n_b == sim.iters_used() <= 5
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= 1e-6 and rel(ctx.positions() - sc.pos, xo - sc.pos) <= 1e-6


def test_defaults_are_the_literal_loop():
    sc = scenes.make("bar3k")
    ctx = mgpbd.Context.from_scene(sc)
    ctx.step(sc.dt, 4)
    st = ctx.stats()
    assert st.n_b == 4 and st.omega_relax == sc.omega_relax


@pytest.mark.parametrize("name", ["bar3k", "block_small"])
def test_pcg_tolerance_exit(name):
    """pcg_tol > 0: the device freezes MGPCG at the first iteration k with ||r_k|| <= pcg_tol ||b||
    (the oracle breaks there) — identical hierarchies, fp64."""
    sc = scenes.make(name)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    import scipy.sparse as sp
    n = r.shape[0] - 1
    A = sp.csr_matrix((v, c, r), shape=(n, n))
    b = A @ np.random.default_rng(3).normal(size=n)      # in the range of A: the residual decreases
    h = O.Hierarchy(r, c, v)
    res = [np.linalg.norm(b - A @ h.pcg(b, K)[0]) / np.linalg.norm(b) for K in range(0, 8)]
    assert res[6] < min(res[:6])
    tol = np.sqrt(res[6] * min(res[:6]))                  # reached first at K = 6
    ho = O.Hierarchy(r, c, v, O.default_config(pcg_tol=tol))
    xo, _, _ = ho.pcg(b, 30)
    ctx = mgpbd.Context.from_scene(sc, pcg_tol=tol)
    ctx.debug_setup_from(v)
    xg = ctx.debug_pcg(b, 30)
    assert rel(xg, xo) <= 1e-9
    assert np.linalg.norm(b - A @ xg) <= tol * np.linalg.norm(b) * (1 + 1e-9)


@pytest.mark.parametrize("name", ["cloth16", "bar3k"])
def test_absolute_residual_exit_frame(name):
    """Alg. 1 l.12 with the absolute eps of the paper's cloth runs ("||b|| < 1e-4"): both sides
    stop after the same outer iteration and agree on the frame."""
    sc = scenes.make(name)
    probe = O.Sim(sc)
    probe.step(sc.dt, 10)
    nb = probe.b_norms(10)
    eps = 1.001 * nb[:5].min()                          # reached within the first 5 iterations
    ctx = mgpbd.Context.from_scene(sc, residual_abs=eps)
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, residual_abs=eps))
    ctx.step(sc.dt, 10)
    sim.step(sc.dt, 10)
    st = ctx.stats()
    assert st.iters_run == sim.iters_used() <= 5 and st.b_last < eps
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= 1e-6 and rel(ctx.positions() - sc.pos, xo - sc.pos) <= 1e-6


@pytest.mark.parametrize("precision", [0, 1], ids=["fp64", "fp32"])
def test_time_budget_exit_frame(precision):
    """Alg. 1 l.12 "timeBudgetExhausted" (reading c21): a budget below one outer iteration stops after it — equal to the
    oracle's 1-iteration frame — and a budget above the frame keeps every iteration."""
    sc = scenes.make("bar3k")
    tol = 1e-6 if precision == 0 else 1e-3
    ctx = mgpbd.Context.from_scene(sc, precision=precision, time_budget_ms=1e-6)
    ctx.step(sc.dt, 8)
    assert ctx.stats().iters_run == 1
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters))
    sim.step(sc.dt, 1)
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= tol and rel(ctx.positions() - sc.pos, xo - sc.pos) <= tol
    ctx.close()
    ctx = mgpbd.Context.from_scene(sc, precision=precision, time_budget_ms=1e7)
    ctx.step(sc.dt, 8)
    assert ctx.stats().iters_run == 8
    ctx.close()
