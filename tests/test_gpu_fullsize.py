"""Parity at BASELINE.json's full sizes in the launch configuration bench.py times (fp32 storage,
matrix-free level 0 with the TMA row kernel, CUDA graphs, persistent coarse kernel): the oracle cannot
run a 1.7M-tet frame in test time, so it checks what it can compute one by one — the whole CSR pattern,
the assembled A_0 on sampled rows and ||b_0|| at the predicted state (Alg. 1 l.1-6), the setup on the
oracle's own A_0 bits (aggregates and level-1 pattern bit-exact, level-1 values) — plus properties
that hold at any size (bitwise determinism, graph replay == eager, pinned vertices fixed)."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

FULL = ["cloth256", "bar50k", "block1.67M", "cloth2048"]


def predicted(sc):
    """Alg. 1 l.1 (semi-implicit Euler): v += dt g for w > 0, x~ = x + dt v."""
    v = sc.vel.copy()
    free = sc.inv_mass > 0
    v[free] += sc.dt * np.array([0.0, -9.8, 0.0])
    return sc.pos + sc.dt * v


def oracle_state(sc):
    xt = predicted(sc)
    if sc.kind == 2:
        C, g = O.eval_distance(sc.verts, xt, O.rest_distance(sc.verts, sc.rest_pos))
    else:
        C, g = O.eval_arap(sc.verts, xt, O.rest_arap(sc.verts, sc.rest_pos)[0])
    return C, g, sc.compliance / sc.dt ** 2


@pytest.fixture(scope="module", params=FULL)
def full(request):
    sc = scenes.make(request.param)
    rowptr, col = O.pattern(sc.verts, sc.n_verts)
    C, g, at = oracle_state(sc)
    return sc, rowptr, col, C, g, at


def test_fullsize_pattern_assembly_rows_and_rhs(full):
    sc, ro, co, C, g, at = full
    ctx = mgpbd.Context.from_scene(sc, precision=1)          # bench configuration
    ctx.step(sc.dt, 1)                                       # one outer iteration at the predicted state
    r, c, v = ctx.level(0)
    assert np.array_equal(r, ro) and np.array_equal(c, co)   # whole pattern, bit-exact
    rows = np.sort(np.random.default_rng(0).choice(sc.n_cons, size=min(4000, sc.n_cons), replace=False))
    vo = O.assemble_rows(rows, sc.verts, sc.inv_mass, g, at, ro, co)
    for i in rows:
        a, e = ro[i], ro[i + 1]
        scale = np.abs(vo[a:e]).max()
        assert np.abs(v[a:e] - vo[a:e]).max() <= 2e-5 * scale, i      # fp32 h, fp32 products
    bn = ctx.stats().b_norm[0]
    assert abs(bn - np.linalg.norm(C)) <= 1e-5 * np.linalg.norm(C)    # b = -C - at*0
    ctx.close()


def test_fullsize_setup_on_oracle_bits(full):
    sc, ro, co, C, g, at = full
    v0 = O.assemble(sc.verts, sc.inv_mass, g, at, ro, co)
    ctx = mgpbd.Context.from_scene(sc, precision=1)
    ctx.debug_setup_from(v0)
    strong = O.soc(ro, co, v0, 0.1)
    agg, na = O.aggregate(ro, co, v0, strong)
    assert np.array_equal(ctx.aggregates(0), agg)
    P = ctx.prolongator(0)
    r1, c1, v1 = ctx.level(1)
    ro1, co1, vo1 = O.galerkin(ro, co, v0, agg, P, na)       # P^T A P with the device's P
    assert np.array_equal(r1, ro1) and np.array_equal(c1, co1)
    assert np.abs(v1 - vo1).max() <= 1e-5 * np.abs(vo1).max()   # fp32 hot refresh of A_1
    ctx.close()


@pytest.mark.parametrize("name", ["block1.67M"])
def test_fullsize_deterministic_and_graph_replay(name, monkeypatch):
    sc = scenes.make(name)
    outs = []
    for env in (None, None, "1"):
        if env:
            monkeypatch.setenv("MGPBD_NO_GRAPH", env)
        ctx = mgpbd.Context.from_scene(sc, precision=1)
        ctx.step(sc.dt, sc.n_iters)
        outs.append((ctx.positions(), ctx.lambdas()))
        ctx.close()
    for x, lam in outs[1:]:
        assert np.array_equal(x, outs[0][0]) and np.array_equal(lam, outs[0][1])
    pinned = sc.inv_mass == 0
    assert np.array_equal(outs[0][0][pinned], sc.pos[pinned])


def test_fullsize_two_virtual_ranks_match_one_context():
    """The row-partitioned path at full size (block1.67M fp32, two virtual ranks on one GPU: halo
    exchange, TMA row kernel from a non-zero first row, replicated coarse kernels) against one context."""
    import threading
    sc = scenes.make("block1.67M")
    ctx = mgpbd.Context.from_scene(sc, precision=1)
    ctx.step(sc.dt, 4)
    x1, l1 = ctx.positions(), ctx.lambdas()
    ctx.close()
    group = mgpbd.VirtualGroup(2)
    out, errs = [None, None], []

    def worker(rank):
        try:
            c = mgpbd.Context.from_scene(sc, precision=1, rank=rank, world=2, vgroup=group)
            c.step(sc.dt, 4)
            out[rank] = (c.positions(), c.lambdas(), c.stats().halo_rows)
            c.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(900)
    assert not errs, errs
    for x, lam, halo in out:
        assert halo > 0
        assert np.linalg.norm(lam - l1) <= 1e-3 * np.linalg.norm(l1)
        assert np.linalg.norm((x - sc.pos) - (x1 - sc.pos)) <= 1e-3 * np.linalg.norm(x1 - sc.pos)
    assert np.array_equal(out[0][1], out[1][1])


@pytest.fixture(scope="module")
def block_oracle_hierarchy():
    sc = scenes.make("block1.67M")
    ro, co = O.pattern(sc.verts, sc.n_verts)
    C, g, at = oracle_state(sc)
    v0 = O.assemble(sc.verts, sc.inv_mass, g, at, ro, co)
    return sc, ro, co, v0, O.Hierarchy(ro, co, v0)       # ~1 min of oracle setup on one core


@pytest.mark.parametrize("precision,tol_v", [(1, 1e-4), (0, 1e-10)])
def test_fullsize_vcycle_and_pcg_on_oracle_hierarchy(block_oracle_hierarchy, precision, tol_v):
    """block1.67M: the whole setup on the oracle's A_0 bits (levels, omegas) and the V-cycle / 5-step
    MGPCG of the device hierarchy (resident coarse kernel, cooperative coarsest inverse) against the
    oracle's, in fp32 (the bench configuration) and fp64."""
    sc, ro, co, v0, h = block_oracle_hierarchy
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.debug_setup_from(v0)
    st = ctx.stats()
    assert st.n_levels == h.n_levels
    for l in range(h.n_levels - 1):
        assert st.n[l] == h.level_size(l)[0]
        assert np.isclose(st.omega[l], h.omega(l), rtol=1e-9), l
    b = np.random.default_rng(0).normal(size=sc.n_cons)
    zg, zo = ctx.debug_vcycle(b), h.vcycle(b)
    assert np.linalg.norm(zg - zo) <= tol_v * np.linalg.norm(zo)
    xg, (xo, rc, _) = ctx.debug_pcg(b, 5), h.pcg(b, 5)
    assert rc == 0 and np.linalg.norm(xg - xo) <= 100 * tol_v * np.linalg.norm(xo)
    ctx.close()
