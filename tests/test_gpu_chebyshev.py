"""GPU parity of the Chebyshev smoother (reading c20)
against the oracle, through the C-ABI: V-cycle / PCG on identical hierarchies, whole frames (fp64 and
fp32, both level-0 operators, with and without the persistent coarse kernel), and sweeps 1..3."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

NAMES = ["cloth16", "cloth64", "bar3k", "block_small"]


def make_scene(name):
    if name == "cloth64":
        return scenes.cloth(64, dt=3e-3, n_iters=5)
    return scenes.make(name)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def ocfg(sc, **kw):
    return O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, smoother=1, **kw)


@pytest.mark.parametrize("sweeps", [1, 2, 3])
@pytest.mark.parametrize("name", ["bar3k", "block_small"])
def test_chebyshev_vcycle_pcg_identical_hierarchy(name, sweeps):
    sc = make_scene(name)
    sim = O.Sim(sc)
    sim.step(sc.dt, 1)
    r, c, v = sim.A()
    h = O.Hierarchy(r, c, v, O.default_config(smoother=1, smoother_sweeps=sweeps))
    ctx = mgpbd.Context.from_scene(sc, smoother=1, smoother_sweeps=sweeps)
    ctx.debug_setup_from(v)
    b = np.random.default_rng(0).normal(size=sc.n_cons)
    assert rel(ctx.debug_vcycle(b), h.vcycle(b)) <= 1e-11
    for K in (1, 5):
        xo, rc, _ = h.pcg(b, K)
        assert rc == 0 and rel(ctx.debug_pcg(b, K), xo) <= 1e-9, K


@pytest.mark.parametrize("op", [0, 1], ids=["csr", "matfree"])
@pytest.mark.parametrize("name", NAMES)
def test_chebyshev_frame_fp64(name, op):
    sc = make_scene(name)
    ctx = mgpbd.Context.from_scene(sc, smoother=1, level0_operator=op)
    sim = O.Sim(sc, ocfg(sc))
    ctx.step(sc.dt, sc.n_iters)
    sim.step(sc.dt, sc.n_iters)
    xo, vo, lo = sim.state()
    assert ctx.stats().indefinite_events == sim.indefinite_events()
    assert rel(ctx.lambdas(), lo) <= 1e-6 and rel(ctx.positions() - sc.pos, xo - sc.pos) <= 1e-6


@pytest.mark.parametrize("name", NAMES)
def test_chebyshev_frame_fp32(name):
    sc = make_scene(name)
    ctx = mgpbd.Context.from_scene(sc, smoother=1, precision=1)
    sim = O.Sim(sc, ocfg(sc))
    ctx.step(sc.dt, sc.n_iters)
    sim.step(sc.dt, sc.n_iters)
    xo, _, lo = sim.state()
    assert rel(ctx.lambdas(), lo) <= 1e-3 and rel(ctx.positions() - sc.pos, xo - sc.pos) <= 1e-3


@pytest.mark.parametrize("sweeps", [1, 3])
def test_chebyshev_per_level_kernels_equal_coarse_kernel(sweeps, monkeypatch):
    """The persistent coarse V-cycle and the per-level kernels apply the same Chebyshev steps."""
    sc = scenes.make("block_small")
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("MGPBD_NO_COARSE_KERNEL", env)
        else:
            monkeypatch.delenv("MGPBD_NO_COARSE_KERNEL", raising=False)
        ctx = mgpbd.Context.from_scene(sc, smoother=1, smoother_sweeps=sweeps)
        ctx.step(sc.dt, 3)
        outs.append(ctx.lambdas())
        ctx.close()
    assert rel(outs[0], outs[1]) <= 1e-9
    sim = O.Sim(sc, ocfg(sc, smoother_sweeps=sweeps))
    sim.step(sc.dt, 3)
    assert rel(outs[0], sim.state()[2]) <= 1e-6


def test_chebyshev_config_errors():
    sc = scenes.make("cloth16")
    for kw in (dict(smoother=2), dict(smoother=1, cheb_lower=1.5), dict(smoother_sweeps=9)):
        with pytest.raises(mgpbd.MgpbdError):
            mgpbd.Context.from_scene(sc, **kw)
