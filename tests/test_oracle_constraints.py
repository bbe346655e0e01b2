"""Pins of the oracle's hash, constraints, pattern, assembly, rhs and update (SURVEY.md §8(c) a1, a2,
a12).  Every check compares the oracle with something other than itself: a published value, a
closed form, a dense brute force, finite differences or a library routine."""
import json
import os

import numpy as np
import pytest
import scipy.linalg

from paper_2505_13390_b200 import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_splitmix64_reference_vectors(O):
    g = GOLD["splitmix64_seed0_first3"]
    inc = int(g["increment"], 16)
    state = 0
    for out in g["outputs"]:
        state = (state + inc) & 0xFFFFFFFFFFFFFFFF
        assert O.mix64(state) == int(out, 16)


def test_hash_uniform_matches_generator_module(O):
    # the input module's numpy hash and the oracle's C hash are independent implementations
    idx = np.arange(1000)
    u_py = scenes.hash_uniform(1, 3, 2, idx)
    u_c = np.array([O.uniform(1, 3, 2, int(i)) for i in idx])
    assert np.array_equal(u_py, u_c)
    assert 0.0 < u_c.min() and u_c.max() < 1.0 and abs(u_c.mean() - 0.5) < 0.05


def test_distance_examples(O):
    for c in GOLD["distance"]["cases"]:
        x = np.array([c["xa"], c["xb"]], float)
        Cv, g = O.eval_distance(np.array([[0, 1]]), x, np.array([c["L"]]))
        assert Cv[0] == c["C"]
        assert g[0, 0].tolist() == c["ga"] and g[0, 1].tolist() == c["gb"]


def test_distance_gradient_finite_differences(O):
    rng = np.random.default_rng(0)
    x = rng.normal(size=(20, 3))
    verts = rng.integers(0, 20, size=(40, 2)).astype(np.int32)
    verts = verts[verts[:, 0] != verts[:, 1]]
    L = rng.uniform(0.5, 2.0, size=verts.shape[0])
    Cv, g = O.eval_distance(verts, x, L)
    eps = 1e-6
    for j in range(verts.shape[0]):
        for s in range(2):
            for r in range(3):
                xp = x.copy(); xm = x.copy()
                xp[verts[j, s], r] += eps; xm[verts[j, s], r] -= eps
                fd = (O.eval_distance(verts[j:j + 1], xp, L[j:j + 1])[0][0] -
                      O.eval_distance(verts[j:j + 1], xm, L[j:j + 1])[0][0]) / (2 * eps)
                assert abs(fd - g[j, s, r]) <= 1e-5, (j, s, r)


def _random_rotation(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q @ np.diag(np.sign(np.diag(r)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def test_polar_special_cases_and_library(O):
    assert np.allclose(O.polar(np.eye(3)), np.eye(3), atol=1e-14)
    assert np.allclose(O.polar(2 * np.eye(3)), np.eye(3), atol=1e-14)
    assert np.array_equal(O.polar(np.zeros((3, 3))), np.eye(3))
    rng = np.random.default_rng(1)
    for _ in range(50):
        Q = _random_rotation(rng)
        S = rng.normal(size=(3, 3)); S = S @ S.T + 0.5 * np.eye(3)
        F = Q @ S
        R = O.polar(F)
        Rl, _ = scipy.linalg.polar(F)            # library polar decomposition
        assert np.allclose(R, Q, atol=1e-9) and np.allclose(R, Rl, atol=1e-9)
    for _ in range(50):                          # inverted elements: det F < 0
        F = rng.normal(size=(3, 3))
        if np.linalg.det(F) > 0:
            F[:, 0] = -F[:, 0]
        R = O.polar(F)
        U, s, Vt = np.linalg.svd(F)              # library SVD, smallest-sigma column flipped
        D = np.eye(3); D[2, 2] = np.sign(np.linalg.det(U @ Vt))
        assert np.allclose(R, U @ D @ Vt, atol=1e-9)
        assert abs(np.linalg.det(R) - 1) < 1e-12 and np.allclose(R.T @ R, np.eye(3), atol=1e-12)


def _one_tet():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) * 0.3
    return np.array([[0, 1, 2, 3]], np.int32), X


def test_arap_rest_rotation_and_stretch_closed_forms(O):
    verts, X = _one_tet()
    Dm, vol = O.rest_arap(verts, X)
    assert np.isclose(vol[0], 0.3 ** 3 / 6)
    Cv, g = O.eval_arap(verts, X, Dm)                      # rest: F = R = I
    assert abs(Cv[0]) < 1e-28 and np.abs(g).max() < 1e-13
    rng = np.random.default_rng(2)
    Q = _random_rotation(rng)
    Cv, g = O.eval_arap(verts, X @ Q.T + 1.0, Dm)          # rigid motion
    assert abs(Cv[0]) < 1e-20 and np.abs(g).max() < 1e-9
    s = np.array([1.3, 0.8, 1.1])                          # F = diag(s): C = sum (s_i - 1)^2
    Cv, g = O.eval_arap(verts, X * s, Dm)
    assert np.isclose(Cv[0], ((s - 1) ** 2).sum(), rtol=1e-12)


def test_arap_gradient_finite_differences_and_translation(O):
    rng = np.random.default_rng(3)
    sc = scenes.make("bar_small")
    Dm, _ = O.rest_arap(sc.verts, sc.rest_pos)
    x = sc.rest_pos + 0.01 * rng.normal(size=sc.rest_pos.shape)
    sub = np.arange(0, sc.n_cons, 7)
    verts = sc.verts[sub]
    Cv, g = O.eval_arap(verts, x, Dm[sub])
    assert np.abs(g.sum(1)).max() < 1e-9 * max(1.0, np.abs(g).max())   # sum_k g_k = 0
    eps = 1e-7
    for j in range(0, len(sub), 3):
        for s_ in range(4):
            for r in range(3):
                xp = x.copy(); xm = x.copy()
                xp[verts[j, s_], r] += eps; xm[verts[j, s_], r] -= eps
                fd = (O.eval_arap(verts[j:j + 1], xp, Dm[sub][j:j + 1])[0][0] -
                      O.eval_arap(verts[j:j + 1], xm, Dm[sub][j:j + 1])[0][0]) / (2 * eps)
                assert abs(fd - g[j, s_, r]) <= 1e-4 * max(1e-3, np.abs(g[j]).max())


def test_lattice_volume_and_masses(O):
    sc = scenes.kuhn_block(10, 2, 2, 0.1, squash=1.0, twist_deg=0.0)
    _, vol = O.rest_arap(sc.verts, sc.rest_pos)
    assert np.isclose(vol.sum(), 10 * 2 * 2 * 0.1 ** 3, rtol=1e-12)
    assert sc.n_cons == 6 * 10 * 2 * 2 and sc.n_verts == 11 * 3 * 3


def _brute_pattern(verts):
    m = verts.shape[0]
    sets = [set(v) for v in verts.tolist()]
    rows = []
    for i in range(m):
        rows.append([j for j in range(m) if j != i and sets[i] & sets[j]] + [i])
    return rows


@pytest.mark.parametrize("name", ["cloth4", "bar_small"])
def test_pattern_vs_bruteforce(O, name):
    sc = scenes.cloth(4) if name == "cloth4" else scenes.make(name)
    rowptr, col = O.pattern(sc.verts, sc.n_verts)
    rows = _brute_pattern(sc.verts)
    assert rowptr[-1] == sum(len(r) for r in rows)
    for i, r in enumerate(rows):
        assert col[rowptr[i]:rowptr[i + 1]].tolist() == r       # sorted off-diagonals, diag last


def test_cloth_counts():
    for N, m in [(1, 5), (2, 16), (16, 800), (256, 197120)]:
        assert scenes.cloth_edges(N).shape[0] == m == 3 * N * N + 2 * N


def _dense_A(sc, g, alpha_tilde):
    m, k = sc.verts.shape
    J = np.zeros((m, 3 * sc.n_verts))
    for j in range(m):
        for s in range(k):
            J[j, 3 * sc.verts[j, s]:3 * sc.verts[j, s] + 3] += g[j, s]
    Minv = np.repeat(sc.inv_mass, 3)
    return (J * Minv) @ J.T + np.diag(alpha_tilde), J


def test_single_edge_assembly(O):
    verts = np.array([[0, 1]], np.int32)
    x = np.array([[0, 0, 0], [1.5, 0, 0]], float)
    Cv, g = O.eval_distance(verts, x, np.array([1.0]))
    rowptr, col = O.pattern(verts, 2)
    val = O.assemble(verts, np.ones(2), g, np.zeros(1), rowptr, col)
    assert val.tolist() == [GOLD["assembly_single_edge"]["A"]]


@pytest.mark.parametrize("name", ["cloth4", "bar_small"])
def test_assembly_vs_dense_bruteforce(O, name):
    sc = scenes.cloth(4, dt=0.02) if name == "cloth4" else scenes.make(name)
    rng = np.random.default_rng(4)
    x = sc.pos + 0.02 * rng.normal(size=sc.pos.shape) * (0.25 if sc.kind == 2 else 0.05)
    if sc.kind == 2:
        Cv, g = O.eval_distance(sc.verts, x, O.rest_distance(sc.verts, sc.rest_pos))
    else:
        Cv, g = O.eval_arap(sc.verts, x, O.rest_arap(sc.verts, sc.rest_pos)[0])
    at = sc.compliance / sc.dt ** 2
    rowptr, col = O.pattern(sc.verts, sc.n_verts)
    val = O.assemble(sc.verts, sc.inv_mass, g, at, rowptr, col)
    A = np.zeros((sc.n_cons, sc.n_cons))
    for i in range(sc.n_cons):
        A[i, col[rowptr[i]:rowptr[i + 1]]] = val[rowptr[i]:rowptr[i + 1]]
    Ad, J = _dense_A(sc, g, at)
    assert np.abs(A - Ad).max() <= 1e-12 * np.abs(Ad).max()
    assert np.array_equal(A, A.T)                        # bitwise symmetric (canonical order)
    np.linalg.cholesky(A)                                # SPD since alpha_tilde > 0
    if sc.kind == 2:                                     # PAPER.md:265 distance: A_ii = w_a + w_b + at
        d = val[rowptr[1:] - 1]
        wsum = sc.inv_mass[sc.verts].sum(1)
        assert np.allclose(d, wsum + at, rtol=1e-13)
    # rhs and apply_dx (Eq. 3, Eq. 5) vs dense
    lam = rng.normal(size=sc.n_cons)
    b = O.rhs(Cv, at, lam)
    assert np.array_equal(b, -Cv - at * lam)
    dl = rng.normal(size=sc.n_cons)
    dx = O.apply_dx(sc.verts, sc.n_verts, sc.inv_mass, g, dl)
    assert np.allclose(dx.ravel(), np.repeat(sc.inv_mass, 3) * (J.T @ dl), rtol=1e-12, atol=1e-300 + 1e-13 * np.abs(dx).max())


def test_rhs_examples(O):
    for c in GOLD["rhs"]["cases"]:
        assert O.rhs(np.array([c["C"]], float), np.array([c["at"]], float), np.array([c["lam"]], float))[0] == c["b"]


def test_compliance_examples():
    # alpha_tilde = 1/(mu V dt^2): input preparation, checked against the SPEC
    for c in GOLD["compliance"]["cases"]:
        assert np.isclose(1.0 / (c["mu"] * c["V"]) / c["dt"] ** 2, c["at"], rtol=1e-12)
