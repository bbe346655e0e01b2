"""Pins of the oracle's V-cycle, MGPCG and Algorithm-1 frame."""
import json
import os

import numpy as np
import pytest

from paper_2505_13390_b200 import scenes
from _util import csr_from_dense_diaglast, dense

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


@pytest.fixture(scope="module")
def bar_sys(O):
    sc = scenes.make("bar3k")
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    return r, c, v, dense(r, c, v)


def test_single_level_vcycle_is_dense_solve(O):
    sc = scenes.make("bar_small")                      # 96 rows < 400: one level (c7)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    h = O.Hierarchy(r, c, v)
    assert h.n_levels == 1
    b = np.random.default_rng(0).normal(size=96)
    A = dense(r, c, v)
    assert np.allclose(h.vcycle(b), np.linalg.solve(A, b), rtol=1e-10)
    x, rc, _ = h.pcg(b, 1)                              # exact after one PCG iteration
    assert rc == 0 and np.allclose(x, np.linalg.solve(A, b), rtol=1e-9)


def test_vcycle_linear_symmetric_zero(O, bar_sys):
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v)
    assert h.n_levels >= 2
    rng = np.random.default_rng(1)
    n = A.shape[0]
    assert np.array_equal(h.vcycle(np.zeros(n)), np.zeros(n))
    for _ in range(10):
        u, w = rng.normal(size=n), rng.normal(size=n)
        a, b = rng.normal(size=2)
        lhs = h.vcycle(a * u + b * w)
        rhs = a * h.vcycle(u) + b * h.vcycle(w)
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(lhs)
        Mu, Mw = h.vcycle(u), h.vcycle(w)
        assert abs(Mu @ w - u @ Mw) <= 1e-8 * abs(Mu @ w) + 1e-8 * np.linalg.norm(Mu) * np.linalg.norm(w) * 1e-3
        assert u @ Mu > 0                                                           # SPD preconditioner


def test_vcycle_two_level_matches_dense_definition(O, bar_sys):
    """Dense re-derivation of one two-level V-cycle from the level matrices and P."""
    r, c, v, A = bar_sys
    cfg = O.default_config(max_levels=2)
    h = O.Hierarchy(r, c, v, cfg)
    assert h.n_levels == 2
    n = A.shape[0]
    agg, P, w = h.agg(0), h.P(0), h.omega(0)
    Pm = np.zeros((n, agg.max() + 1)); Pm[np.arange(n), agg] = P
    Ac = Pm.T @ A @ Pm
    Dinv = 1.0 / np.diag(A)
    b = np.random.default_rng(2).normal(size=n)
    x = np.zeros(n)
    for _ in range(2):
        x = x + w * Dinv * (b - A @ x)
    x = x + Pm @ np.linalg.solve(Ac, Pm.T @ (b - A @ x))
    for _ in range(2):
        x = x + w * Dinv * (b - A @ x)
    assert np.allclose(h.vcycle(b), x, rtol=1e-9, atol=1e-12 * np.abs(x).max())


def test_pcg_finite_termination_and_monotone_A_norm(O, bar_sys):
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v)
    b = np.random.default_rng(3).normal(size=A.shape[0])
    xs = np.linalg.solve(A, b)
    errs = []
    for K in range(1, 41, 3):
        x, rc, _ = h.pcg(b, K)
        assert rc == 0
        e = x - xs
        errs.append(np.sqrt(e @ A @ e))
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-9) for i in range(len(errs) - 1))   # monotone in A-norm
    x, rc, _ = h.pcg(b, 300)
    assert np.linalg.norm(A @ x - b) <= 1e-3 * np.linalg.norm(b)
    # CG finite termination on a tiny SPD system forced into several levels (K >> n): dense solution
    sc = scenes.make("bar_small")
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    A = dense(r, c, v)
    h = O.Hierarchy(r, c, v, O.default_config(min_coarse=20))
    assert h.n_levels >= 2
    b = np.random.default_rng(5).normal(size=A.shape[0])
    x, rc, _ = h.pcg(b, 400)
    assert np.linalg.norm(A @ x - b) <= 1e-8 * np.linalg.norm(b)


def test_pcg_identity(O):
    r, c, v = csr_from_dense_diaglast(np.eye(500))    # all-singleton stall => one dense level
    h = O.Hierarchy(r, c, v)
    b = np.random.default_rng(4).normal(size=500)
    x, rc, _ = h.pcg(b, 1)
    assert rc == 0 and np.allclose(x, b, rtol=1e-14)


def _python_frame(O, sc, n_iters, omega, gravity=(0, -9.8, 0), backtrack=False, omega_min=1e-3, tol=0.0,
                  trace=None):
    """Algorithm 1 with a dense direct solve in place of MGPCG; optional backtracking
    (halve omega when ||b|| rises) and the ||b|| < tol ||b_0|| exit (l.12)."""
    x = sc.pos.copy(); v = sc.vel.copy(); w = sc.inv_mass
    x_old = x.copy()
    v[w > 0] += sc.dt * np.asarray(gravity)
    x = x + sc.dt * v
    lam = np.zeros(sc.n_cons)
    at = sc.compliance / sc.dt ** 2
    rowptr, col = O.pattern(sc.verts, sc.n_verts)
    rest = O.rest_distance(sc.verts, sc.rest_pos) if sc.kind == 2 else O.rest_arap(sc.verts, sc.rest_pos)[0]
    bprev = None
    for ite in range(n_iters):
        Cv, g = (O.eval_distance if sc.kind == 2 else O.eval_arap)(sc.verts, x, rest)
        A = dense(rowptr, col, O.assemble(sc.verts, w, g, at, rowptr, col))
        b = -Cv - at * lam
        nb = np.linalg.norm(b)
        if ite == 0:
            b0 = nb
        if backtrack and bprev is not None and nb > bprev:
            omega = max(0.5 * omega, omega_min)
        bprev = nb
        dl = np.linalg.solve(A, b)
        dx = O.apply_dx(sc.verts, sc.n_verts, w, g, dl)
        lam += dl
        x = x + omega * dx
        if trace is not None:
            trace.append((ite, nb, omega))
        if tol > 0 and nb < tol * b0:
            break
    return x, (x - x_old) / sc.dt, lam


@pytest.mark.parametrize("name", ["cloth4", "bar_small"])
def test_frame_equals_dense_direct_frame(O, name):
    sc = scenes.cloth(4, dt=3e-3) if name == "cloth4" else scenes.make(name)
    cfg = O.default_config(omega_relax=sc.omega_relax, pcg_iters=3)
    sim = O.Sim(sc, cfg)
    assert sim.step(sc.dt, 4) == 0
    x, v, lam = sim.state()
    xr, vr, lr = _python_frame(O, sc, 4, sc.omega_relax)
    assert np.allclose(lam, lr, rtol=1e-9, atol=1e-12 * np.abs(lr).max())
    assert np.allclose(x - sc.pos, xr - sc.pos, rtol=1e-9, atol=1e-12 * np.abs(xr - sc.pos).max())
    # Alg. 1 l.17: v = (x - x_old)/dt, against the dense-direct frame's own velocity
    assert np.allclose(v, vr, rtol=1e-9, atol=1e-12 * np.abs(vr).max())


def test_single_constraint_closed_form_eq4_eq5(O):
    """One distance constraint: the hierarchy is one 1x1 level, so each outer iteration is exactly
    Eq. 4 (dlambda = -(C + at lambda)/(w_a + w_b + at)) followed by Eq. 5."""
    g = GOLD["single_constraint_xpbd"]
    X = np.array([[0, 0, 0], [1, 0, 0]], float)
    x0 = np.array([[0, 0, 0], [2, 0, 0]], float)          # stretch 1
    sc = scenes.Scene("edge", 2, np.array([[0, 1]], np.int32), X, x0, np.zeros_like(X),
                      np.ones(2), np.zeros(1), 1.0, 1.0)
    cfg = O.default_config(omega_relax=1.0, gravity=(0, 0, 0), pcg_iters=1)
    sim = O.Sim(sc, cfg)
    sim.step(1.0, 1)
    x, v, lam = sim.state()
    assert np.isclose(lam[0], g["dlambda"], rtol=1e-15)
    assert np.allclose(x, [[g["move"], 0, 0], [2 - g["move"], 0, 0]], rtol=1e-15)
    # compliant case, two iterations, omega = 0.5, masses (1, 3)
    alpha, dt, om = 0.3, 0.5, 0.5
    sc = scenes.Scene("edge", 2, np.array([[0, 1]], np.int32), X, x0, np.zeros_like(X),
                      np.array([1.0, 1 / 3.0]), np.array([alpha]), dt, om)
    sim = O.Sim(sc, O.default_config(omega_relax=om, gravity=(0, 0, 0), pcg_iters=2))
    sim.step(dt, 2)
    x, _, lam = sim.state()
    at = alpha / dt ** 2
    xa, xb, l = x0[0].copy(), x0[1].copy(), 0.0
    for _ in range(2):
        d = xa - xb; L = np.linalg.norm(d); u = d / L
        dl = -((L - 1.0) + at * l) / (1.0 + 1 / 3.0 + at)           # Eq. 4
        xa = xa + om * 1.0 * u * dl; xb = xb - om * (1 / 3.0) * u * dl   # Eq. 5
        l += dl
    assert np.isclose(lam[0], l, rtol=1e-13) and np.allclose(x, [xa, xb], rtol=1e-13)


def test_rest_state_identity_and_pins(O):
    for sc in [scenes.cloth(8, jitter=0.0), scenes.kuhn_block(4, 2, 2, 0.05, squash=1.0, twist_deg=0.0, jitter=0.0)]:
        cfg = O.default_config(omega_relax=sc.omega_relax, gravity=(0, 0, 0))
        sim = O.Sim(sc, cfg)
        sim.step(sc.dt, 3)
        x, v, lam = sim.state()
        assert np.abs(x - sc.pos).max() <= 1e-12 and np.abs(lam).max() <= 1e-9
    sc = scenes.cloth(8)
    sim = O.Sim(sc)
    for _ in range(3):
        sim.step(sc.dt, 3)
    x, v, _ = sim.state()
    pinned = sc.inv_mass == 0
    assert np.array_equal(x[pinned], sc.pos[pinned]) and np.all(v[pinned] == 0)


def test_semi_euler_free_fall(O):
    g = GOLD["semi_euler"]
    X = np.array([[0, 0, 0], [1, 0, 0]], float)
    sc = scenes.Scene("edge", 2, np.array([[0, 1]], np.int32), X, X.copy(), np.zeros_like(X),
                      np.ones(2), np.array([1e300]), g["dt"], 1.0)
    sim = O.Sim(sc, O.default_config(omega_relax=0.0))
    sim.step(g["dt"], 1)
    x, _, _ = sim.state()
    assert np.allclose(x - X, [[0, g["dy"], 0]] * 2, rtol=1e-12)


def test_lambda_fixed_point(O):
    """At convergence of the outer loop lambda = -alpha_tilde^-1 C."""
    sc = scenes.cloth(4, dt=0.02, stiffness=1e3)
    sim = O.Sim(sc, O.default_config(omega_relax=1.0, pcg_iters=5, gravity=(0, -9.8, 0)))
    sim.step(sc.dt, 60)
    x, _, lam = sim.state()
    Cv, _ = O.eval_distance(sc.verts, x, O.rest_distance(sc.verts, sc.rest_pos))
    at = sc.compliance / sc.dt ** 2
    assert np.allclose(lam, -Cv / at, rtol=1e-6, atol=1e-9 * np.abs(lam).max())


def test_deterministic(O):
    sc = scenes.make("cloth16")
    outs = []
    for _ in range(2):
        sim = O.Sim(sc)
        sim.step(sc.dt, sc.n_iters)
        outs.append(sim.state())
    assert all(np.array_equal(a, b) for a, b in zip(*outs))


# ------------------------------------------------------------------ Chebyshev smoother (reading c20)
def _cheb_T(k, z):
    return np.cos(k * np.arccos(z)) if abs(z) <= 1 else np.cosh(k * np.arccosh(abs(z))) * np.sign(z) ** k


def _tridiag(n, c):
    A = np.eye(n) - c * (np.eye(n, k=1) + np.eye(n, k=-1))
    return A, 1.0 - 2.0 * c * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))


@pytest.mark.parametrize("sweeps", [1, 2, 3])
def test_chebyshev_residual_is_the_scaled_chebyshev_polynomial(O, sweeps):
    """A = tridiag(-c, 1, -c) has D = I and eigenpairs (1 - 2c cos(k pi/(n+1)), sin).  From x = 0 with
    b = an eigenvector v (eigenvalue lam), s Chebyshev steps on [lo, hi] leave the residual
    T_s((theta - lam)/delta) / T_s(theta/delta) * v — the defining property of the Chebyshev iteration
    (Saad, Alg. 12.1) — and the interval is hi = safety * lambda_max(D^-1 A), lo = 0.25 hi (c20)."""
    n, c = 500, 0.45
    A, lam = _tridiag(n, c)
    r, cc, v = csr_from_dense_diaglast(A)
    cfg = O.default_config(smoother=1, smoother_sweeps=sweeps, power_iters=3000)
    h = O.Hierarchy(r, cc, v, cfg)
    assert h.n_levels >= 2
    theta, delta = h.cheb(0)
    hi, lo = theta + delta, theta - delta
    # power method from below, tiny spectral gap at the top: 1e-3 (its own pin is in test_oracle_setup)
    assert 0 <= 1.1 * lam.max() - hi <= 1e-3 * hi and abs(lo - 0.25 * hi) <= 1e-12 * hi
    i = np.arange(1, n + 1)
    for k in (1, 7, 60, 250, 499):
        vk = np.sin(k * i * np.pi / (n + 1))
        x = h.smooth(0, vk, np.zeros(n))
        res = vk - A @ x
        want = _cheb_T(sweeps, (theta - lam[k - 1]) / delta) / _cheb_T(sweeps, theta / delta)
        assert np.allclose(res, want * vk, rtol=1e-9, atol=1e-11), k


def test_chebyshev_one_step_is_jacobi_with_one_over_theta(O):
    """s = 1: x = D^-1 b / theta (the Chebyshev iteration's first step is damped Jacobi)."""
    n = 500
    A, _ = _tridiag(n, 0.3)
    A = A * np.linspace(1.0, 3.0, n)[:, None] ** 0.5 * np.linspace(1.0, 3.0, n)[None, :] ** 0.5  # D != I
    r, c, v = csr_from_dense_diaglast(A)
    h = O.Hierarchy(r, c, v, O.default_config(smoother=1, smoother_sweeps=1))
    theta, _ = h.cheb(0)
    b = np.random.default_rng(4).normal(size=n)
    assert np.allclose(h.smooth(0, b, np.zeros(n)), b / np.diag(A) / theta, rtol=1e-14)


def test_chebyshev_vcycle_linear_symmetric_and_pcg(O, bar_sys):
    """The Chebyshev V-cycle is a symmetric positive definite linear operator (identical pre/post
    polynomials in D^-1 A) and MGPCG with it converges."""
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v, O.default_config(smoother=1))
    rng = np.random.default_rng(6)
    n = A.shape[0]
    for _ in range(5):
        u, w = rng.normal(size=n), rng.normal(size=n)
        a, bb = rng.normal(size=2)
        lhs = h.vcycle(a * u + bb * w)
        assert np.linalg.norm(lhs - a * h.vcycle(u) - bb * h.vcycle(w)) <= 1e-10 * np.linalg.norm(lhs)
        Mu, Mw = h.vcycle(u), h.vcycle(w)
        assert abs(Mu @ w - u @ Mw) <= 1e-9 * np.linalg.norm(Mu) * np.linalg.norm(w)
        assert u @ Mu > 0
    b = rng.normal(size=n)
    x, rc, _ = h.pcg(b, 300)
    assert rc == 0 and np.linalg.norm(A @ x - b) <= 1e-3 * np.linalg.norm(b)


def test_chebyshev_two_level_matches_dense_definition(O, bar_sys):
    """Dense re-derivation of a two-level Chebyshev V-cycle: x_{k+1} = x_k + d_k with
    d_0 = D^-1 r_0 / theta, d_k = rho_k rho_{k-1} d_{k-1} + 2 rho_k / delta D^-1 r_k."""
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v, O.default_config(max_levels=2, smoother=1))
    n = A.shape[0]
    agg, P = h.agg(0), h.P(0)
    theta, delta = h.cheb(0)
    Pm = np.zeros((n, agg.max() + 1)); Pm[np.arange(n), agg] = P
    Ac = Pm.T @ A @ Pm
    Dinv = 1.0 / np.diag(A)

    def cheb(x, b):
        sigma = theta / delta
        rho = 1 / sigma
        d = Dinv * (b - A @ x) / theta
        x = x + d
        rho_new = 1 / (2 * sigma - rho)
        d = rho_new * rho * d + 2 * rho_new / delta * Dinv * (b - A @ x)
        return x + d

    b = np.random.default_rng(7).normal(size=n)
    x = cheb(np.zeros(n), b)
    x = x + Pm @ np.linalg.solve(Ac, Pm.T @ (b - A @ x))
    x = cheb(x, b)
    assert np.allclose(h.vcycle(b), x, rtol=1e-9, atol=1e-12 * np.abs(x).max())


# ------------------------------------------------------------------ outer-loop variants (reading c21)
def test_backtrack_rule_examples(O):
    """decrease -> unchanged; increase halves; repeated halving floors at 1e-3."""
    omega, seq = 0.1, []
    for _ in range(9):
        omega = max(0.5 * omega, 1e-3)
        seq.append(omega)
    assert seq[6] == 1e-3 and seq[5] > 1e-3 and seq[-1] == 1e-3


@pytest.mark.parametrize("name", ["cloth4", "bar_small"])
def test_backtracking_and_residual_exit_equal_dense_frame(O, name):
    """Backtracking omega and the ||b|| < eps exit in the oracle's frame against the dense Python
    Algorithm 1 (single-level hierarchy: MGPCG is exact), and the halving actually triggered."""
    sc = scenes.cloth(4, dt=3e-3) if name == "cloth4" else scenes.make(name)
    om = 1.0 if name == "cloth4" else 0.9         # large omega: overshoot, ||b|| rises, halving kicks in
    cfg = O.default_config(omega_relax=om, pcg_iters=3, backtrack=1)
    sim = O.Sim(sc, cfg)
    assert sim.step(sc.dt, 12) == 0
    trace = []
    xr, _, lr = _python_frame(O, sc, 12, om, backtrack=True, trace=trace)
    x, _, lam = sim.state()
    # 12 outer iterations of a stiff system amplify the solves' rounding (Cholesky vs LAPACK): 1e-7
    assert np.abs(lam - lr).max() <= 1e-7 * np.abs(lr).max()
    assert np.abs((x - sc.pos) - (xr - sc.pos)).max() <= 1e-7 * np.abs(xr - sc.pos).max()
    assert sim.omega() == trace[-1][2] < om                      # halved at least once
    nb = sim.b_norms(12)
    assert np.allclose(nb, [t[1] for t in trace], rtol=1e-7)
    # residual exit: stops at the first iteration whose ||b|| < tol ||b_0||, after its update
    tol = 1.001 * nb[:6].min() / nb[0]
    cfg = O.default_config(omega_relax=om, pcg_iters=3, backtrack=1, residual_tol=tol)
    sim = O.Sim(sc, cfg)
    sim.step(sc.dt, 12)
    trace = []
    xr, _, lr = _python_frame(O, sc, 12, om, backtrack=True, tol=tol, trace=trace)
    assert sim.iters_used() == len(trace) < 12
    assert np.abs(sim.state()[2] - lr).max() <= 1e-7 * np.abs(lr).max()


# ------------------------------------------------------------------ multicolour GS smoother (reading c22)
def test_gs_sweep_is_the_permuted_triangular_solve(O, bar_sys):
    """One forward multicolour GS sweep = solve (D + L_p) x' = b - U_p x in the (colour, index) order;
    the backward (post) sweep = (D + U_p) x' = b - L_p x (the order reversed)."""
    import scipy.linalg as sl
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v, O.default_config(smoother=2, smoother_sweeps=1))
    colours, _ = O.colour(r, c)
    order = np.lexsort((np.arange(A.shape[0]), colours))        # by colour, then index
    Ap = A[np.ix_(order, order)]
    rng = np.random.default_rng(8)
    b, x0 = rng.normal(size=A.shape[0]), rng.normal(size=A.shape[0])
    Lw, Up = np.tril(Ap), np.triu(Ap, 1)
    want = np.empty_like(b)
    want[order] = sl.solve_triangular(Lw, b[order] - Up @ x0[order], lower=True)
    assert np.allclose(h.smooth(0, b, x0), want, rtol=1e-10, atol=1e-12 * np.abs(want).max())
    Uw, Lp = np.triu(Ap), np.tril(Ap, -1)
    want[order] = sl.solve_triangular(Uw, b[order] - Lp @ x0[order], lower=False)
    assert np.allclose(h.smooth(0, b, x0, post=True), want, rtol=1e-10, atol=1e-12 * np.abs(want).max())


def test_gs_vcycle_symmetric_positive_and_pcg(O, bar_sys):
    """Forward pre-sweeps and reversed post-sweeps make the GS V-cycle a symmetric positive definite
    preconditioner (identical pre- and post-smoothers keep the cycle symmetric)."""
    r, c, v, A = bar_sys
    h = O.Hierarchy(r, c, v, O.default_config(smoother=2))
    rng = np.random.default_rng(9)
    n = A.shape[0]
    for _ in range(5):
        u, w = rng.normal(size=n), rng.normal(size=n)
        Mu, Mw = h.vcycle(u), h.vcycle(w)
        assert abs(Mu @ w - u @ Mw) <= 1e-9 * np.linalg.norm(Mu) * np.linalg.norm(w)
        assert u @ Mu > 0
    b = rng.normal(size=n)
    x, rc, _ = h.pcg(b, 300)
    assert rc == 0 and np.linalg.norm(A @ x - b) <= 1e-3 * np.linalg.norm(b)


def test_pcg_tolerance_exit(O, bar_sys):
    """pcg_tol > 0 (off by default, reading c10): MGPCG stops before the first
    iteration k with ||r_k|| <= pcg_tol ||b|| — the result equals the fixed-count solve truncated at
    that k, and meets the tolerance."""
    r, c, v, A = bar_sys
    n = A.shape[0]
    b = A @ np.random.default_rng(11).normal(size=n)     # in the range of A: the residual decreases
    h = O.Hierarchy(r, c, v)
    res = [np.linalg.norm(b - A @ h.pcg(b, K)[0]) / np.linalg.norm(b) for K in range(0, 41)]
    assert res[8] < min(res[:8])
    tol = np.sqrt(res[8] * min(res[:8]))
    K = next(k for k in range(41) if res[k] <= tol)
    assert K == 8
    ht = O.Hierarchy(r, c, v, O.default_config(pcg_tol=tol))
    xt, _, _ = ht.pcg(b, 40)
    assert np.array_equal(xt, h.pcg(b, K)[0])
    assert np.linalg.norm(b - A @ xt) <= tol * np.linalg.norm(b) * (1 + 1e-12)


def test_setup_schedule_literal_and_resetup_on_indefinite(O):
    """Alg. 1 l.7: setup at ite 0 of frames with frame % setup_interval == 0.  With
    resetup_on_indef = 0 (the literal paper) nothing else triggers it, even after PCG iterations with
    <z,r> <= 0; with resetup_on_indef = 1 (reading c13 extension) a frame with such events is followed by
    a setup.  bar3k with lambda_safety = 1 (literal omega) has events from frame 0 on."""
    sc = scenes.make("bar3k")
    ev, su = {}, {}
    for re in (0, 1):
        cfg = O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, lambda_safety=1.0,
                               resetup_on_indef=re)
        sim = O.Sim(sc, cfg)
        ev[re], su[re] = [], []
        for _ in range(4):
            sim.step(sc.dt, sc.n_iters)
            ev[re].append(sim.indefinite_events()); su[re].append(sim.setups())
    assert sum(ev[0]) > 0 and su[0] == [1, 1, 1, 1]
    for f in range(1, 4):
        assert su[1][f] - su[1][f - 1] == (1 if ev[1][f - 1] > 0 else 0)
    assert su[1][-1] > 1


def test_time_budget_exit(O):
    """Alg. 1 l.12 "timeBudgetExhausted" (reading c21): a budget every iteration exceeds stops the frame
    after its first outer iteration — the frame then equals a 1-iteration frame — and a budget none reaches leaves
    the fixed-count frame unchanged."""
    from paper_2505_13390_b200 import scenes
    sc = scenes.make("bar_small")
    base = dict(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters)
    one = O.Sim(sc, O.default_config(**base))
    assert one.step(sc.dt, 1) == 0
    tiny = O.Sim(sc, O.default_config(time_budget_ms=1e-9, **base))
    assert tiny.step(sc.dt, 6) == 0 and tiny.iters_used() == 1
    for a, b in zip(tiny.state(), one.state()):
        assert np.array_equal(a, b)
    full = O.Sim(sc, O.default_config(**base))
    huge = O.Sim(sc, O.default_config(time_budget_ms=1e9, **base))
    assert full.step(sc.dt, 6) == 0 and huge.step(sc.dt, 6) == 0 and huge.iters_used() == 6
    for a, b in zip(huge.state(), full.state()):
        assert np.array_equal(a, b)
