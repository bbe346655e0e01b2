"""Pins of the oracle's k > 1 near-kernel variant ("We repeat this six
times to generate six distinct B"; "R of QR decomposition serves as B at the next level";
readings c23-c25 in DESIGN.md §2): k bootstrapped columns, per-aggregate thin QR injection with
rank-deficient aggregates, general Galerkin P^T A P, and the k = 6 hierarchy / V-cycle / frame."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2505_13390_b200 import scenes
from _util import csr_from_dense_diaglast, dense


def pdense(P, n, nc):
    r, c, v = P
    M = np.zeros((n, nc))
    for i in range(n):
        M[i, c[r[i]:r[i + 1]]] = v[r[i]:r[i + 1]]
    return M


@pytest.fixture(scope="module")
def bar_sys(O):
    sc = scenes.make("bar3k")
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    return r, c, v


def test_bootstrap_k_columns(O, bar_sys):
    """Column 0 is the k = 1 bootstrap bit for bit; column c is 3 GS sweeps (forward substitution in
    (colour, index) order, scipy) from x_0[i] = U(stream 3, 0, i + c n) max|A_ij| (reading c23)."""
    r, c, v = bar_sys
    n = r.shape[0] - 1
    col, _ = O.colour(r, c, 1)
    B = O.gs_bootstrap_k(r, c, v, col, 4, sweeps=3, seed=1)
    assert B.shape == (n, 4)
    assert np.array_equal(B[:, 0], O.gs_bootstrap(r, c, v, col, sweeps=3, seed=1))
    A = sp.csr_matrix(dense(r, c, v))
    perm = np.lexsort((np.arange(n), col))
    Ap = A[perm][:, perm]
    Lw = sp.tril(Ap, 0, format="csr"); Up = sp.triu(Ap, 1, format="csr")
    for cc in range(4):
        x = (scenes.hash_uniform(1, 3, 0, np.arange(n) + cc * n) * np.abs(v).max())[perm]
        for _ in range(3):
            x = spla.spsolve_triangular(Lw, -(Up @ x), lower=True)
        assert np.allclose(B[perm, cc], x, rtol=1e-10, atol=1e-12 * np.abs(x).max()), cc
    # distinct columns, each an algebraically smooth vector after 20 sweeps
    B20 = O.gs_bootstrap_k(r, c, v, col, 6, sweeps=20, seed=1)
    for cc in range(6):
        x0 = scenes.hash_uniform(1, 3, 0, np.arange(n) + cc * n) * np.abs(v).max()
        assert np.linalg.norm(A @ B20[:, cc]) / np.linalg.norm(B20[:, cc]) <= 0.1 * np.linalg.norm(A @ x0) / np.linalg.norm(x0)
    assert np.linalg.matrix_rank(B20, tol=1e-8 * np.abs(B20).max()) == 6


def test_prolongator_qr_k1_reduces_to_normalisation(O):
    rng = np.random.default_rng(0)
    agg = rng.integers(0, 7, 40).astype(np.int32); agg[:7] = np.arange(7)
    B = rng.normal(size=40)
    P1, Bn1 = O.prolongator(agg, 7, B)
    (pr, pc, pv), Bn, coff = O.prolongator_qr(agg, 7, B[:, None])
    assert np.array_equal(pr, np.arange(41)) and np.array_equal(pc, agg) and np.array_equal(coff, np.arange(8))
    assert np.allclose(pv, P1, rtol=1e-14) and np.allclose(Bn[:, 0], Bn1, rtol=1e-14)


def test_prolongator_qr_full_rank_against_numpy_qr(O):
    """P^T P = I, P B_next = B, and per aggregate Q, R equal numpy.linalg.qr's up to column signs (R
    diagonal > 0 fixes them)."""
    rng = np.random.default_rng(1)
    n, na, k = 60, 5, 3
    agg = np.repeat(np.arange(na), n // na).astype(np.int32)
    rng.shuffle(agg)
    B = rng.normal(size=(n, k))
    P, Bn, coff = O.prolongator_qr(agg, na, B)
    assert np.array_equal(coff, np.arange(0, k * na + 1, k))
    Pm = pdense(P, n, na * k)
    assert np.allclose(Pm.T @ Pm, np.eye(na * k), atol=1e-12)
    assert np.allclose(Pm @ Bn, B, atol=1e-12 * np.abs(B).max())
    for a in range(na):
        mem = np.flatnonzero(agg == a)
        Qn, Rn = np.linalg.qr(B[mem])
        s = np.sign(np.diag(Rn))
        Qn, Rn = Qn * s, Rn * s[:, None]
        assert np.allclose(Pm[mem][:, coff[a]:coff[a + 1]], Qn, atol=1e-12)
        assert np.allclose(Bn[coff[a]:coff[a + 1]], Rn, atol=1e-12 * np.abs(Rn).max())
        R = Bn[coff[a]:coff[a + 1]]
        assert np.all(np.diag(R) > 0) and np.allclose(np.tril(R, -1), 0.0)


def test_prolongator_qr_rank_deficient_aggregates(O):
    """Readings c24/c25: an aggregate smaller than k keeps |N_a| columns, linearly dependent columns are
    dropped (their R entries hold the projections, so P B_next = B still holds), a zero block gets the
    uniform column with a zero R row; P keeps orthonormal columns (full column rank)."""
    rng = np.random.default_rng(2)
    k = 6
    sizes = [2, 8, 8, 5]                      # agg 0: 2 members < k
    agg = np.concatenate([np.full(s, a) for a, s in enumerate(sizes)]).astype(np.int32)
    n = agg.shape[0]
    B = rng.normal(size=(n, k))
    m1 = agg == 1
    B[m1, 3] = 2.0 * B[m1, 0] - B[m1, 1]     # agg 1: column 3 in the span of columns 0, 1
    B[agg == 2] = 0.0                         # agg 2: zero block
    P, Bn, coff = O.prolongator_qr(agg, len(sizes), B)
    r_a = np.diff(coff)
    assert list(r_a) == [2, 5, 1, 5]
    Pm = pdense(P, n, coff[-1])
    assert np.allclose(Pm.T @ Pm, np.eye(coff[-1]), atol=1e-12)
    assert np.allclose(Pm @ Bn, B, atol=1e-10 * np.abs(B).max())
    assert np.allclose(Pm[agg == 2, coff[2]], 1 / np.sqrt(8)) and np.all(Bn[coff[2]] == 0.0)
    # the dropped column keeps its projections: R row entries for column 3 of agg 1 = (2, -1, 0, ...) R
    R1 = Bn[coff[1]:coff[2]]
    assert np.allclose(R1[:, 3], 2.0 * R1[:, 0] - R1[:, 1], atol=1e-12 * np.abs(R1).max())


def test_galerkin_general_p_against_dense_and_k1(O):
    rng = np.random.default_rng(5)
    from test_oracle_setup import random_spd_pattern
    for t in range(6):
        n = int(rng.integers(30, 150)); na = int(rng.integers(2, n // 8 + 2)); k = int(rng.integers(1, 5))
        A = random_spd_pattern(n, 3, 300 + t)
        r, c, v = csr_from_dense_diaglast(A)
        agg = rng.integers(0, na, n).astype(np.int32); agg[:na] = np.arange(na)
        P, Bn, coff = O.prolongator_qr(agg, na, rng.normal(size=(n, k)))
        nc = int(coff[-1])
        cr, cc, cv = O.galerkin_p(r, c, v, P, nc)
        Pm = pdense(P, n, nc)
        Ad = Pm.T @ A @ Pm
        Ac = dense(cr, cc, cv)
        assert np.abs(Ac - Ad).max() <= 1e-12 * np.abs(Ad).max()
        for I in range(nc):                                   # diag last, off-diagonals ascending
            row = cc[cr[I]:cr[I + 1]]
            assert row[-1] == I and np.all(np.diff(row[:-1]) > 0)
        np.linalg.cholesky(Ac)                                # SPD: P has orthonormal columns
        if k == 1:                                            # same order as the k = 1 product: bitwise
            cr1, cc1, cv1 = O.galerkin(r, c, v, agg, P[2], na)
            assert np.array_equal(cr1, cr) and np.array_equal(cc1, cc) and np.array_equal(cv1, cv)


@pytest.fixture(scope="module")
def bar_hier_k6(O, bar_sys):
    r, c, v = bar_sys
    cfg = O.default_config(k_nullspace=6, min_coarse=50)
    return (r, c, v), O.Hierarchy(r, c, v, cfg)


def test_hierarchy_k6_invariants(O, bar_hier_k6):
    (r, c, v), h = bar_hier_k6
    assert h.n_levels >= 3
    B0 = h.B0()
    assert B0.shape == (r.shape[0] - 1, 6)
    for l in range(h.n_levels - 1):
        n, _ = h.level_size(l)
        nc, _ = h.level_size(l + 1)
        P = h.P_csr(l)
        Pm = pdense(P, n, nc)
        assert np.allclose(Pm.T @ Pm, np.eye(nc), atol=1e-10)
        Al = dense(*h.level(l))
        Ac = dense(*h.level(l + 1))
        assert np.abs(Ac - Pm.T @ Al @ Pm).max() <= 1e-12 * np.abs(Ac).max()
        np.linalg.cholesky(Ac)
        assert 0 < h.omega(l) < 2
    # level 0: P B_1 = B_0 (R of QR is the next level's B) on full-rank aggregates
    n0, _ = h.level_size(0)
    agg = h.agg(0)
    assert np.bincount(agg).min() >= 6


def test_vcycle_k6_two_level_dense_and_symmetric(O, bar_sys):
    r, c, v = bar_sys
    A = dense(r, c, v)
    n = A.shape[0]
    h = O.Hierarchy(r, c, v, O.default_config(k_nullspace=6, max_levels=2))
    assert h.n_levels == 2
    nc, _ = h.level_size(1)
    Pm = pdense(h.P_csr(0), n, nc)
    Ac = Pm.T @ A @ Pm
    Dinv = 1.0 / np.diag(A)
    w = h.omega(0)
    b = np.random.default_rng(2).normal(size=n)
    x = np.zeros(n)
    for _ in range(2):
        x = x + w * Dinv * (b - A @ x)
    x = x + Pm @ np.linalg.solve(Ac, Pm.T @ (b - A @ x))
    for _ in range(2):
        x = x + w * Dinv * (b - A @ x)
    assert np.allclose(h.vcycle(b), x, rtol=1e-9, atol=1e-12 * np.abs(x).max())
    rng = np.random.default_rng(3)
    u, z = rng.normal(size=n), rng.normal(size=n)
    Mu, Mz = h.vcycle(u), h.vcycle(z)
    assert abs(Mu @ z - u @ Mz) <= 1e-8 * abs(Mu @ z) and u @ Mu > 0


def test_frame_k6_with_exact_pcg_equals_dense_direct_frame(O):
    """With pcg_iters >= m, MGPCG is exact (CG finite termination) whatever the preconditioner, so a k = 6
    frame equals the dense-direct Algorithm 1."""
    from test_oracle_solve import _python_frame
    sc = scenes.cloth(6, dt=3e-3, stiffness=1e3)      # moderate kappa: CG reaches the exact solve
    cfg = O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.n_cons + 5, k_nullspace=6, min_coarse=20)
    sim = O.Sim(sc, cfg)
    assert sim.step(sc.dt, 3) == 0
    assert sim.hierarchy().n_levels >= 2
    x, v, lam = sim.state()
    xr, vr, lr = _python_frame(O, sc, 3, sc.omega_relax)
    assert np.allclose(lam, lr, rtol=1e-7, atol=1e-9 * np.abs(lr).max())
    assert np.allclose(x - sc.pos, xr - sc.pos, rtol=1e-7, atol=1e-9 * np.abs(xr - sc.pos).max())
