"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element on identical
seeded inputs.  Tolerances: patterns, aggregates, colour-independent integer
results bit-exact; fp64 values <= 1e-12 relative per stage on identical inputs; whole frame fp64
<= 1e-6 relative, fp32 <= 1e-3 relative (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

SMALL = ["cloth16", "bar_small", "bar3k", "cloth64", "block_small"]


def make_scene(name):
    if name == "cloth64":
        return scenes.cloth(64, dt=3e-3, n_iters=5)
    return scenes.make(name)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def ctx_for(sc, precision=0, **kw):
    return mgpbd.Context.from_scene(sc, precision=precision, **kw)


@pytest.mark.parametrize("name", SMALL)
def test_pattern_bit_exact(name):
    sc = make_scene(name)
    ctx = ctx_for(sc)
    r, c, _ = ctx.level(0)
    ro, co = O.pattern(sc.verts, sc.n_verts)
    assert np.array_equal(r, ro) and np.array_equal(c, co)


@pytest.mark.parametrize("name", SMALL)
def test_assembly_and_rhs_fp64(name):
    sc = make_scene(name)
    ctx = ctx_for(sc)
    ctx.step(sc.dt, 1)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = ctx.level(0)
    ro, co, vo = sim.A()
    assert np.array_equal(r, ro) and np.array_equal(c, co)
    scale = np.abs(vo).max()
    assert np.abs(v - vo).max() <= 1e-12 * scale
    # bitwise symmetric (canonical shared-vertex order on the device as well)
    n = r.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(r))
    import scipy.sparse as sp
    A = sp.csr_matrix((v, (rows, c)), shape=(n, n))
    assert (A != A.T).nnz == 0
    st = ctx.stats()
    assert np.isclose(st.b_norm[0], sim.b_norms(1)[0], rtol=1e-12)


def oracle_setup(sc, ctx=None):
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    return r, c, v, O.Hierarchy(r, c, v)


@pytest.mark.parametrize("name", SMALL)
def test_setup_identical_input_bits(name):
    """Setup on the oracle's own A_0 bits: aggregates and patterns bit-exact, P/B/omega/levels to 1e-12."""
    sc = make_scene(name)
    r, c, v, h = oracle_setup(sc)
    ctx = ctx_for(sc)
    ctx.debug_setup_from(v)
    st = ctx.stats()
    assert st.n_levels == h.n_levels
    if h.n_levels > 1:
        assert st.n_colours == h.n_colours
        assert rel(ctx.near_kernel(), h.B0()) <= 1e-10
    for l in range(h.n_levels):
        rg, cg, vg = ctx.level(l)
        ro, co, vo = h.level(l)
        assert np.array_equal(rg, ro) and np.array_equal(cg, co), l
        assert np.abs(vg - vo).max() <= 1e-12 * np.abs(vo).max(), l
        if l + 1 < h.n_levels:
            assert np.array_equal(ctx.aggregates(l), h.agg(l)), l
            assert np.abs(ctx.prolongator(l) - h.P(l)).max() <= 1e-12, l
            assert np.isclose(st.omega[l], h.omega(l), rtol=1e-10), l


@pytest.mark.parametrize("name", SMALL)
def test_vcycle_and_pcg_identical_hierarchy(name):
    sc = make_scene(name)
    r, c, v, h = oracle_setup(sc)
    ctx = ctx_for(sc)
    ctx.debug_setup_from(v)
    rng = np.random.default_rng(0)
    b = rng.normal(size=sc.n_cons)
    assert rel(ctx.debug_vcycle(b), h.vcycle(b)) <= 1e-11
    for K in (1, 3, 10):
        xg = ctx.debug_pcg(b, K)
        xo, rc, _ = h.pcg(b, K)
        assert rc == 0
        assert rel(xg, xo) <= 1e-9, K


@pytest.mark.parametrize("op", [0, 1], ids=["csr", "matfree"])
@pytest.mark.parametrize("name", SMALL)
def test_frame_fp64(name, op):
    sc = make_scene(name)
    ctx = ctx_for(sc, level0_operator=op)
    sim = O.Sim(sc)
    ctx.step(sc.dt, sc.n_iters)
    assert sim.step(sc.dt, sc.n_iters) == 0
    xo, vo, lo = sim.state()
    xg, vg, lg = ctx.positions(), ctx.velocities(), ctx.lambdas()
    assert rel(lg, lo) <= 1e-6
    assert rel(xg - sc.pos, xo - sc.pos) <= 1e-6 and rel(xg, xo) <= 1e-6
    assert rel(vg, vo) <= 1e-6
    st = ctx.stats()
    assert np.allclose(st.b_norm[:sc.n_iters], sim.b_norms(sc.n_iters), rtol=1e-6)
    assert st.indefinite_events == sim.indefinite_events()


@pytest.mark.parametrize("name", SMALL)
def test_matrix_free_vcycle_and_pcg(name):
    """Matrix-free level 0 (A x = H(H^T x) + at x from the scaled gradients) inside
    the V-cycle and MGPCG, against the oracle's assembled-CSR hierarchy at the same state."""
    sc = make_scene(name)
    ctx = ctx_for(sc, level0_operator=1)
    ctx.step(sc.dt, 1)                      # one outer iteration: setup and h at the same state
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    h = O.Hierarchy(r, c, v)
    rng = np.random.default_rng(1)
    b = rng.normal(size=sc.n_cons)
    assert rel(ctx.debug_vcycle(b), h.vcycle(b)) <= 1e-10
    for K in (1, 5):
        xo, rc, _ = h.pcg(b, K)
        assert rc == 0 and rel(ctx.debug_pcg(b, K), xo) <= 1e-8, K


@pytest.mark.parametrize("name", ["bar3k", "cloth64", "block_small"])
def test_galerkin_from_gradients_level1(name):
    """With the matrix-free level 0 the Eq. 6 refresh of A_1 = P^T A_0 P is computed from the scaled
    gradients (vertex-aggregate sums, csrc/vagal.cu); it must equal the oracle's explicit product."""
    sc = make_scene(name)
    ctx = ctx_for(sc, level0_operator=1)
    ctx.step(sc.dt, 1)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    h = O.Hierarchy(r, c, v)
    assert h.n_levels > 1
    rg, cg, vg = ctx.level(1)
    ro, co, vo = h.level(1)
    assert np.array_equal(rg, ro) and np.array_equal(cg, co)
    assert np.abs(vg - vo).max() <= 1e-12 * np.abs(vo).max()


@pytest.mark.parametrize("name", ["cloth64", "bar3k", "block_small"])
def test_setup_galerkin_vertex_aggregate_equals_csr(name, monkeypatch):
    """In matrix-free mode the setup's A_1 = P^T A_0 P (pattern and fp64 values) comes from the gradients
    (csrc/vagal.cu va_coarse_pattern + va_numeric) instead of the CSR Galerkin plan; the hierarchy it
    builds must be the one the CSR product builds (MGPBD_NO_VA_SETUP=1)."""
    sc = make_scene(name)
    out = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("MGPBD_NO_VA_SETUP", "1")
        ctx = ctx_for(sc, level0_operator=1)
        ctx.step(sc.dt, 1)   # setup at the first outer iteration, then the hot refreshes
        nl = ctx.stats().n_levels
        out.append((nl, [ctx.aggregates(l) for l in range(nl - 1)], [ctx.level(l) for l in range(1, nl)]))
        ctx.close()
    (n0, a0, m0), (n1, a1, m1) = out
    assert n0 == n1 and n0 > 1
    for x, y in zip(a0, a1):
        assert np.array_equal(x, y)
    for (r0_, c0_, v0_), (r1_, c1_, v1_) in zip(m0, m1):
        assert np.array_equal(r0_, r1_) and np.array_equal(c0_, c1_)
        assert np.abs(v0_ - v1_).max() <= 1e-12 * np.abs(v1_).max()


@pytest.mark.parametrize("precision", [0, 1])
def test_matrix_free_equals_csr_frames(precision):
    sc = scenes.make("block_small")
    outs = []
    for op in (0, 1):
        ctx = ctx_for(sc, precision=precision, level0_operator=op)
        ctx.step(sc.dt, sc.n_iters)
        outs.append((ctx.positions() - sc.pos, ctx.lambdas()))
        ctx.close()
    tol = 1e-9 if precision == 0 else 1e-3
    assert rel(outs[1][0], outs[0][0]) <= tol and rel(outs[1][1], outs[0][1]) <= tol


def test_bar3k_multiframe_indefinite_resetup_fp64():
    """The bar-twist release drifts lambda_max(D^-1 A) past the lazily-set omega; both sides detect
    <z,r> <= 0 identically and re-run the setup at the next frame (reading c13)."""
    sc = scenes.make("bar3k")
    ctx = ctx_for(sc)
    sim = O.Sim(sc)
    ctx.step(sc.dt, 20)
    sim.step(sc.dt, 20)
    assert ctx.stats().indefinite_events == sim.indefinite_events() == 0
    xo, _, lo = sim.state()      # before any event: element-wise parity
    assert rel(ctx.lambdas(), lo) <= 1e-6 and rel(ctx.positions() - sc.pos, xo - sc.pos) <= 1e-6
    ctx.step(sc.dt, 20)
    sim.step(sc.dt, 20)
    # an indefinite CG step amplifies rounding differences, so after it only the event is compared
    assert ctx.stats().indefinite_events > 0 and sim.indefinite_events() > 0
    ctx.step(sc.dt, 20)
    assert ctx.stats().setup_ran == 1      # early re-setup (frame 2 is not a multiple of 20)


@pytest.mark.parametrize("op", [0, 1], ids=["csr", "matfree"])
@pytest.mark.parametrize("name", SMALL)
def test_frame_fp32(name, op):
    sc = make_scene(name)
    ctx = ctx_for(sc, precision=1, level0_operator=op)
    sim = O.Sim(sc)
    ctx.step(sc.dt, sc.n_iters)
    sim.step(sc.dt, sc.n_iters)
    xo, _, lo = sim.state()
    xg, lg = ctx.positions(), ctx.lambdas()
    assert rel(lg, lo) <= 1e-3
    assert rel(xg - sc.pos, xo - sc.pos) <= 1e-3


def test_three_frames_lazy_setup_and_stale():
    sc = scenes.make("cloth16")
    ctx = ctx_for(sc, setup_interval=2)
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, setup_interval=2))
    ran = []
    for f in range(3):
        ctx.step(sc.dt, 4)
        sim.step(sc.dt, 4)
        ran.append(ctx.stats().setup_ran)
    assert ran == [1, 0, 1]
    ctx.setup_hierarchy(); sim.mark_stale()
    ctx.step(sc.dt, 4); sim.step(sc.dt, 4)
    assert ctx.stats().setup_ran == 1
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= 1e-6 and rel(ctx.positions(), xo) <= 1e-6


def test_single_constraint_closed_form():
    X = np.array([[0, 0, 0], [1, 0, 0]], float)
    x0 = np.array([[0, 0, 0], [2, 0, 0]], float)
    ctx = mgpbd.Context(2, np.array([[0, 1]], np.int32), X, np.ones(2), np.zeros(1), pos=x0,
                        omega_relax=1.0, gravity=(0, 0, 0), pcg_iters=1)
    ctx.step(1.0, 1)
    assert np.isclose(ctx.lambdas()[0], -0.5, rtol=1e-15)            # Eq. 4
    assert np.allclose(ctx.positions(), [[0.5, 0, 0], [1.5, 0, 0]], rtol=1e-15)   # Eq. 5


def test_rest_state_and_pins():
    sc = scenes.cloth(8, jitter=0.0)
    ctx = ctx_for(sc, gravity=(0, 0, 0))
    ctx.step(sc.dt, 3)
    assert np.abs(ctx.positions() - sc.pos).max() <= 1e-12
    sc = scenes.make("bar3k")
    ctx = ctx_for(sc)
    for _ in range(2):
        ctx.step(sc.dt, 3)
    pinned = sc.inv_mass == 0
    assert np.array_equal(ctx.positions()[pinned], sc.pos[pinned])


@pytest.mark.parametrize("precision", [0, 1])
def test_deterministic(precision):
    sc = scenes.make("bar3k")
    outs = []
    for _ in range(2):
        ctx = ctx_for(sc, precision=precision)
        ctx.step(sc.dt, 3)
        outs.append((ctx.positions(), ctx.lambdas()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("precision", [0, 1])
def test_graph_replay_equals_eager(precision, monkeypatch):
    """The captured CUDA graphs replay exactly the eager launch sequence (bitwise)."""
    sc = scenes.make("block_small")
    outs = []
    for no_graph in ("1", None):
        if no_graph:
            monkeypatch.setenv("MGPBD_NO_GRAPH", "1")
        else:
            monkeypatch.delenv("MGPBD_NO_GRAPH", raising=False)
        ctx = ctx_for(sc, precision=precision, setup_interval=2)
        for _ in range(3):
            ctx.step(sc.dt, 4)
        outs.append((ctx.positions(), ctx.lambdas()))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_step_argument_errors():
    sc = scenes.make("cloth16")
    ctx = ctx_for(sc)
    with pytest.raises(mgpbd.MgpbdError):
        ctx.step(0.0, 1)
    with pytest.raises(mgpbd.MgpbdError):
        ctx.step(sc.dt, 0)
    with pytest.raises(mgpbd.MgpbdError):
        ctx.aggregates(0)          # no hierarchy before the first step


@pytest.mark.parametrize("precision", [0, 1])
def test_coarse_kernel_variants_agree(precision, monkeypatch):
    """The shared-memory-resident coarse V-cycle (default), the global-memory coarse kernel and the
    per-level kernels apply the same operators (summation order differs only inside restrictions)."""
    sc = scenes.make("block_small")
    outs = []
    for env in ({}, {"MGPBD_NO_RES_COARSE": "1"}, {"MGPBD_NO_COARSE_KERNEL": "1"}):
        for k in ("MGPBD_NO_RES_COARSE", "MGPBD_NO_COARSE_KERNEL"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ctx = ctx_for(sc, precision=precision, setup_interval=2)
        for _ in range(2):
            ctx.step(sc.dt, 4)
        outs.append((ctx.positions() - sc.pos, ctx.lambdas()))
        ctx.close()
    tol = 1e-9 if precision == 0 else 1e-3
    for x, lam in outs[1:]:
        assert rel(x, outs[0][0]) <= tol and rel(lam, outs[0][1]) <= tol


def test_phase_times_cover_the_frame():
    """stats.ms_* (profile = 1): the phases add up to the frame (minus setup and small glue)."""
    sc = scenes.make("block_small")
    ctx = ctx_for(sc, precision=1)
    ctx.set_profiling(True)
    for _ in range(2):
        ctx.step(sc.dt, sc.n_iters)
    st = ctx.stats()
    parts = st.ms_assemble + st.ms_galerkin + st.ms_vcycle + st.ms_pcg_other + st.ms_update
    assert min(st.ms_assemble, st.ms_galerkin, st.ms_vcycle, st.ms_pcg_other, st.ms_update) > 0
    assert 0.6 * (st.ms_frame - st.ms_setup) <= parts <= st.ms_frame - st.ms_setup
    ctx.set_profiling(False)
    ctx.step(sc.dt, sc.n_iters)
    assert ctx.stats().ms_vcycle == 0.0


def test_single_tet_closed_form():
    """One ARAP tetrahedron: A is 1x1, so the first outer iteration is Eq. 4,
    dlambda = -(C + at lambda) / (sum_k w_k |grad_k C|^2 + at), then Eq. 5 — against the oracle."""
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) * 0.1
    x0 = X.copy(); x0[3] += [0.02, -0.01, 0.03]
    w = np.array([0.0, 2.0, 3.0, 4.0])
    comp = np.array([1e-6])
    ctx = mgpbd.Context(4, np.array([[0, 1, 2, 3]], np.int32), X, w, comp, pos=x0, gravity=(0, 0, 0),
                        omega_relax=1.0, pcg_iters=1)
    ctx.step(1e-2, 1)
    Cv, g = O.eval_arap(np.array([[0, 1, 2, 3]], np.int32), x0, O.rest_arap(np.array([[0, 1, 2, 3]], np.int32), X)[0])
    at = comp[0] / 1e-4
    dl = -Cv[0] / ((w[:, None] * g[0] ** 2).sum() + at)
    assert np.isclose(ctx.lambdas()[0], dl, rtol=1e-11)
    assert np.allclose(ctx.positions(), x0 + (w[:, None] * g[0]) * dl, rtol=1e-11, atol=1e-15)


def test_all_pinned_block():
    """Every vertex pinned: A = diag(at), positions never move and lambda = -C / at after one iteration."""
    sc = scenes.make("bar_small")
    w = np.zeros_like(sc.inv_mass)
    ctx = mgpbd.Context(sc.kind, sc.verts, sc.rest_pos, w, sc.compliance, pos=sc.pos, pcg_iters=2)
    ctx.step(sc.dt, 1)
    assert np.array_equal(ctx.positions(), sc.pos)
    Cv, _ = O.eval_arap(sc.verts, sc.pos, O.rest_arap(sc.verts, sc.rest_pos)[0])
    assert np.allclose(ctx.lambdas(), -Cv / (sc.compliance / sc.dt ** 2), rtol=1e-10)


def test_degenerate_rest_tet_rejected():
    X = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 1, 0]], float)   # collinear -> zero volume
    with pytest.raises(mgpbd.MgpbdError):
        mgpbd.Context(4, np.array([[0, 1, 2, 3]], np.int32), X, np.ones(4), np.ones(1))


def test_pass_burst_hook():
    sc = scenes.make("block_small")
    ctx = ctx_for(sc, precision=1)
    with pytest.raises(mgpbd.MgpbdError):
        ctx.pass_burst(4)                      # no state before the first step
    ctx.step(sc.dt, 2)
    ms, by = ctx.pass_burst(8)
    assert ms > 0 and by > 8 * sc.n_cons * 4
    x_before = ctx.positions()
    ctx.step(sc.dt, 2)                         # the context keeps working after the hook
    assert np.isfinite(ctx.positions()).all() and not np.array_equal(ctx.positions(), x_before)


@pytest.mark.parametrize("precision", [0, 1])
def test_tma_and_register_row_kernels_agree(precision, monkeypatch):
    """The TMA-pipelined matrix-free row kernel and the register-streaming one (MGPBD_NO_TMA) compute
    the same rows (only the dot partials' grid differs)."""
    sc = scenes.make("block_small")
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("MGPBD_NO_TMA", env)
        else:
            monkeypatch.delenv("MGPBD_NO_TMA", raising=False)
        ctx = ctx_for(sc, precision=precision)
        ctx.step(sc.dt, 4)
        outs.append((ctx.positions() - sc.pos, ctx.lambdas()))
        ctx.close()
    tol = 1e-9 if precision == 0 else 1e-3
    assert rel(outs[1][0], outs[0][0]) <= tol and rel(outs[1][1], outs[0][1]) <= tol
