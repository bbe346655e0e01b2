"""The north_star target row (BASELINE.json: "a 1.7M-tet synthetic block at 20 AMG-PCG iterations per
frame that matches the oracle within tolerance") and the bench's own hot path at scale.

* mid-size frames (blockslab32: 393,216 rows, 4 levels, 3-4 128-row tiles per TMA CTA) in fp64 and
  fp32 against the oracle, 2-norm and element-wise (max-abs over the max), at 5 outer iterations; the
  7-level hierarchy of the full block is covered by the block1.67M frame below;
* 20-iteration frames against the oracle's own rounding-sensitivity envelope (the fixed-count outer
  iteration amplifies rounding differences exponentially);
* the TMA row kernel's stage ring wrapping on every CTA (grid capped by MGPBD_MF_GRID_CAP) on small frames;
* the block1.67M frame in the bench configuration (fp32 storage, matrix-free level 0 + TMA row kernel,
  gradient Galerkin, CUDA graphs, resident coarse kernel) against the oracle's frame;
* the full-size V-cycle and MGPCG through the hot matrix-free operator (mgpbd_debug_prepare) against the
  oracle's hierarchy built from its own assembly at the same predicted state.
Tolerances: BASELINE.json north_star (fp64 1e-6, fp32 1e-3 relative)."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

FULL_ITERS = 2   # outer iterations of the full-size frame (the oracle needs ~10-20 s per iteration;
                 # fp32 rounding stays below 1e-3 only for the first few iterations, see SLAB_ITERS)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def maxrel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def check_frame(ctx, sim, sc, tol, label):
    xo, vo, lo = sim.state()
    xg, vg, lg = ctx.positions(), ctx.velocities(), ctx.lambdas()
    errs = {"lambda": (rel(lg, lo), maxrel(lg, lo)), "dx": (rel(xg - sc.pos, xo - sc.pos), maxrel(xg - sc.pos, xo - sc.pos)),
            "v": (rel(vg, vo), maxrel(vg, vo))}
    print(label, {k: f"{a:.2e}/{b:.2e}" for k, (a, b) in errs.items()})
    for k, (a, b) in errs.items():
        assert a <= tol and b <= tol, (label, k, a, b)


def predicted(sc):
    """Alg. 1 l.1 (semi-implicit Euler): v += dt g for w > 0, x~ = x + dt v."""
    v = sc.vel.copy()
    v[sc.inv_mass > 0] += sc.dt * np.array([0.0, -9.8, 0.0])
    return sc.pos + sc.dt * v


# Outer iterations of the element-wise comparisons: the fixed-count outer iteration amplifies rounding
# differences ~10x per iteration on the block (reading p1: the oracle perturbed by 1e-15
# moves lambda by 1e-13 after 2, 1e-9 after 5, 4e-3 after 20 iterations on blockslab32), so fp64 is
# compared after 5 iterations and fp32 (unit roundoff 6e-8) after 2; longer frames against the envelope.
SLAB_ITERS = {0: 5, 1: 2}


@pytest.fixture(scope="module")
def slab():
    sc = scenes.make("blockslab32")
    sims = {}
    for p, n in SLAB_ITERS.items():
        sims[p] = O.Sim(sc)
        assert sims[p].step(sc.dt, n) == 0
    return sc, sims


@pytest.mark.parametrize("precision", [0, 1], ids=["fp64", "fp32"])
def test_blockslab32_frame(slab, precision):
    sc, sims = slab
    sim = sims[precision]
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.step(sc.dt, SLAB_ITERS[precision])
    st = ctx.stats()
    h = sim.hierarchy()
    assert st.n_levels == h.n_levels >= 4
    assert [int(st.n[l]) for l in range(st.n_levels)] == [h.level_size(l)[0] for l in range(h.n_levels)]
    assert st.indefinite_events == sim.indefinite_events() == 0
    check_frame(ctx, sim, sc, 1e-6 if precision == 0 else 1e-3, f"blockslab32 fp{'32' if precision else '64'}")
    ctx.close()


def perturbed(sc, eps, seed=0):
    """The same scene with every initial coordinate scaled by (1 + eps U(-1, 1)): a rounding-sized
    perturbation of the input."""
    import copy
    s2 = copy.copy(sc)
    s2.pos = sc.pos * (1.0 + eps * np.random.default_rng(seed).uniform(-1.0, 1.0, sc.pos.shape))
    return s2


@pytest.mark.parametrize("name,precision", [("block_small", 0), ("block_small", 1), ("blockslab32", 0)])
def test_twenty_iteration_frame_within_rounding_envelope(name, precision):
    """At 20 outer iterations the fixed-count Algorithm 1 (10-step MGPCG per iteration) amplifies
    rounding-level input differences by ~1e7-1e12 (reading p1): the oracle itself, with
    its initial positions perturbed by 1e-15 relative, moves lambda by ~1e-4 (block_small) to ~4e-3
    (blockslab32).  So the GPU frame is checked against that envelope: its distance to the oracle must
    not exceed 10x the oracle's distance to its own perturbed run (perturbation = the unit roundoff of
    the GPU's storage precision), and the ||b|| trajectory must match to the same envelope."""
    sc = scenes.make(name)
    eps = 1e-15 if precision == 0 else 1e-7
    a, b = O.Sim(sc), O.Sim(perturbed(sc, eps))
    a.step(sc.dt, 20); b.step(sc.dt, 20)
    _, _, la = a.state()
    _, _, lb = b.state()
    env = rel(lb, la)
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.step(sc.dt, 20)
    dev = rel(ctx.lambdas(), la)
    bn_env = np.abs(b.b_norms(20) / a.b_norms(20) - 1).max()
    bn_dev = np.abs(np.array(ctx.stats().b_norm[:20]) / a.b_norms(20) - 1).max()
    print(f"{name} fp{'32' if precision else '64'} 20 iterations: GPU-oracle {dev:.2e}, oracle envelope {env:.2e}; "
          f"||b|| {bn_dev:.2e} vs {bn_env:.2e}")
    assert dev <= 10 * env + 1e-9 and bn_dev <= 10 * bn_env + 1e-9
    ctx.close()


@pytest.mark.parametrize("precision", [0, 1], ids=["fp64", "fp32"])
@pytest.mark.parametrize("cap", [1, 3, 7])
def test_tma_ring_wraps(monkeypatch, precision, cap):
    """Every TMA row-kernel CTA streams many tiles (the 3-stage ring refills and its mbarrier parity flips
    dozens of times): frames against the oracle and against the uncapped grid."""
    sc = scenes.make("block_small")            # 10,368 rows = 81 tiles of 128
    sim = O.Sim(sc)
    sim.step(sc.dt, sc.n_iters)
    ref = mgpbd.Context.from_scene(sc, precision=precision)
    ref.step(sc.dt, sc.n_iters)
    monkeypatch.setenv("MGPBD_MF_GRID_CAP", str(cap))
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.step(sc.dt, sc.n_iters)
    tol = 1e-6 if precision == 0 else 1e-3
    check_frame(ctx, sim, sc, tol, f"block_small cap {cap}")
    # same operator, different number of dot partials: equal up to the partial-sum order
    assert rel(ctx.lambdas(), ref.lambdas()) <= (1e-10 if precision == 0 else 1e-4)
    ctx.close(); ref.close()


@pytest.fixture(scope="module")
def block_frame():
    sc = scenes.make("block1.67M")
    sim = O.Sim(sc)
    assert sim.step(sc.dt, FULL_ITERS) == 0
    return sc, sim


@pytest.mark.parametrize("precision", [1, 0], ids=["fp32-bench", "fp64"])
def test_target_block_frame(block_frame, precision):
    """Frame 0 of block1.67M with FULL_ITERS outer iterations (setup at ite 0, 10 MGPCG iterations
    each): fp32 is the bench configuration (the default context: matrix-free + TMA, graphs, resident
    coarse kernel); every CTA of the TMA row kernel streams ~15 tiles."""
    sc, sim = block_frame
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.step(sc.dt, FULL_ITERS)
    st = ctx.stats()
    h = sim.hierarchy()
    assert [int(st.n[l]) for l in range(st.n_levels)] == [h.level_size(l)[0] for l in range(h.n_levels)]
    assert st.indefinite_events == sim.indefinite_events()
    assert np.allclose(st.b_norm[:FULL_ITERS], sim.b_norms(FULL_ITERS), rtol=1e-6 if precision == 0 else 1e-3)
    check_frame(ctx, sim, sc, 1e-6 if precision == 0 else 1e-3, f"block1.67M fp{'32' if precision else '64'}")
    ctx.close()


@pytest.fixture(scope="module")
def block_hier():
    """The oracle's hierarchy from its own assembly at the predicted state of frame 0 (Alg. 1 l.1-7)."""
    sc = scenes.make("block1.67M")
    xt = predicted(sc)
    C, g = O.eval_arap(sc.verts, xt, O.rest_arap(sc.verts, sc.rest_pos)[0])
    r, c = O.pattern(sc.verts, sc.n_verts)
    v = O.assemble(sc.verts, sc.inv_mass, g, sc.compliance / sc.dt ** 2, r, c)
    return sc, xt, O.Hierarchy(r, c, v)


@pytest.mark.parametrize("precision", [1, 0], ids=["fp32", "fp64"])
def test_fullsize_matrix_free_vcycle_and_pcg(block_hier, precision):
    sc, xt, h = block_hier
    ctx = mgpbd.Context.from_scene(sc, precision=precision)
    ctx.debug_prepare(sc.dt)
    assert np.abs(ctx.positions() - xt).max() <= 1e-14 * np.abs(xt).max()
    assert np.array_equal(ctx.aggregates(0), h.agg(0))        # same SOC decisions from both assemblies
    assert [ctx.level_size(l)[0] for l in range(h.n_levels)] == [h.level_size(l)[0] for l in range(h.n_levels)]
    b = np.random.default_rng(7).normal(size=sc.n_cons)
    vt = rel(ctx.debug_vcycle(b), h.vcycle(b))
    xo, rc, _ = h.pcg(b, 5)
    pt = rel(ctx.debug_pcg(b, 5), xo)
    print(f"block1.67M matrix-free fp{'32' if precision else '64'}: V-cycle {vt:.2e} 5-step MGPCG {pt:.2e}")
    if precision == 0:
        assert vt <= 1e-9 and pt <= 1e-7
    else:
        assert vt <= 1e-4 and pt <= 1e-2
    ctx.close()
