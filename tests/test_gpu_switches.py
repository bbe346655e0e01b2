"""Every kernel-variant switch selects another implementation of the same operators: a frame
under each switch against the oracle (fp64, 1e-6; reading p1: 3 outer iterations keep the oracle's own rounding
sensitivity far below the bar).  block_small with min_coarse = 30 has 4 levels, so the persistent coarse
kernels, the cluster tail and the coarsest inverse all run."""
import numpy as np
import pytest

import oracle as O
from paper_2505_13390_b200 import mgpbd, scenes

pytestmark = pytest.mark.gpu

MF_SWITCHES = ["", "MGPBD_NO_GRAPH=1", "MGPBD_NO_TMA=1", "MGPBD_NO_RES_COARSE=1", "MGPBD_NO_COARSE_KERNEL=1",
               "MGPBD_COARSE_FROM=2", "MGPBD_NO_GJ_COOP=1", "MGPBD_NO_VA_SETUP=1", "MGPBD_NO_POWER_COOP=1",
               "MGPBD_NO_TAIL=1", "MGPBD_NO_VJ16=1", "MGPBD_NO_V16=1", "MGPBD_VG_TMA=1", "MGPBD_MF_GRID_CAP=2",
               "MGPBD_RES_CAP=4096", "MGPBD_FUSE_J0=1", "MGPBD_NO_FUSED_TAIL=1",
               "MGPBD_TAIL_SCALAR_BCAST=1", "MGPBD_SOLO=1", "MGPBD_SOLO=1 MGPBD_NO_TAIL=1",
               "MGPBD_DENSE_CUT=0", "MGPBD_DENSE_CUT=64", "MGPBD_DENSE_CUT=100000",
               "MGPBD_DENSE_CUT=64 MGPBD_NO_TAIL=1", "MGPBD_DENSE_CUT=64 MGPBD_NO_RES_COARSE=1", "MGPBD_NO_X1_FUSE=1", "MGPBD_FIN_IN_ROWS=1", "MGPBD_NO_VG_PDL=1", "MGPBD_VEC_CPT=1", "MGPBD_RESTRICT_G8=1", "MGPBD_NO_EVAL_HV=1",
               "MGPBD_GJ_BIG_N=0", "MGPBD_TILE_LONG_ROWS=1"]
CSR_SWITCHES = ["", "MGPBD_NO_BAND=1", "MGPBD_NO_ROWS=1", "MGPBD_NO_BAND=1 MGPBD_NO_ROWS=1", "MGPBD_GJ_BIG_N=0"]
ITERS = 3


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def ref():
    sc = scenes.make("block_small")
    sim = O.Sim(sc, O.default_config(omega_relax=sc.omega_relax, pcg_iters=sc.pcg_iters, min_coarse=30))
    assert sim.step(sc.dt, ITERS) == 0
    assert sim.hierarchy().n_levels >= 4
    return sc, sim


def run(monkeypatch, sc, switch, op, precision=0):
    for kv in switch.split():
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    ctx = mgpbd.Context.from_scene(sc, precision=precision, level0_operator=op, min_coarse=30)
    ctx.step(sc.dt, ITERS)
    out = ctx.lambdas(), ctx.positions(), ctx.stats().n_levels
    ctx.close()
    return out


@pytest.mark.parametrize("switch", MF_SWITCHES)
def test_matrix_free_switch(monkeypatch, ref, switch):
    sc, sim = ref
    xo, _, lo = sim.state()
    lg, xg, nl = run(monkeypatch, sc, switch, 1)
    assert nl == sim.hierarchy().n_levels
    assert rel(lg, lo) <= 1e-6 and rel(xg - sc.pos, xo - sc.pos) <= 1e-6, switch


@pytest.mark.parametrize("switch", CSR_SWITCHES)
def test_csr_switch(monkeypatch, ref, switch):
    sc, sim = ref
    xo, _, lo = sim.state()
    lg, xg, _ = run(monkeypatch, sc, switch, 0)
    assert rel(lg, lo) <= 1e-6 and rel(xg - sc.pos, xo - sc.pos) <= 1e-6, switch


@pytest.mark.parametrize("switch", ["", "MGPBD_SOLO=1", "MGPBD_NO_TAIL=1", "MGPBD_NO_FUSED_TAIL=1",
                                    "MGPBD_DENSE_CUT=0", "MGPBD_DENSE_CUT=100000",
                                    "MGPBD_TAIL_SCALAR_BCAST=1",
                                    "MGPBD_NO_VJ16=1 MGPBD_NO_V16=1"])
def test_fp32_switch(monkeypatch, ref, switch):
    sc, sim = ref
    xo, _, lo = sim.state()
    lg, xg, _ = run(monkeypatch, sc, switch, 1, precision=1)
    assert rel(lg, lo) <= 1e-3 and rel(xg - sc.pos, xo - sc.pos) <= 1e-3, switch


@pytest.mark.parametrize("precision,tol", [(0, 1e-12), (1, 1e-4)], ids=["fp64", "fp32"])
def test_dense_bottom_equals_level_by_level_cycle(monkeypatch, precision, tol):
    """Reading c27: the V-cycle whose bottom levels are applied as the explicit sub-cycle matrix M equals the
    level-by-level cycle on the same hierarchy (identical inputs, deterministic setup) up to rounding, for a
    cut at every coarse level (MGPBD_DENSE_CUT rows) and through the resident, global and per-level kernels."""
    sc = scenes.make("block_small")
    rng = np.random.default_rng(7)
    b = rng.normal(size=sc.n_cons)
    out = {}
    for cut in (0, 64, 400, 100000):
        for extra in ("", "MGPBD_NO_RES_COARSE=1", "MGPBD_NO_COARSE_KERNEL=1"):
            monkeypatch.setenv("MGPBD_DENSE_CUT", str(cut))
            for k in ("MGPBD_NO_RES_COARSE", "MGPBD_NO_COARSE_KERNEL"):
                monkeypatch.delenv(k, raising=False)
            if extra:
                monkeypatch.setenv(extra.split("=")[0], "1")
            ctx = mgpbd.Context.from_scene(sc, precision=precision, min_coarse=30)
            ctx.debug_prepare(sc.dt)
            out[(cut, extra)] = (ctx.debug_vcycle(b), ctx.stats().n_levels)
            ctx.close()
    z0, nl = out[(0, "")]
    assert nl >= 4
    for key, (z, n) in out.items():
        assert n == nl
        assert rel(z, z0) <= tol, (key, rel(z, z0))


@pytest.mark.parametrize("precision", [0, 1], ids=["fp64", "fp32"])
@pytest.mark.parametrize("switch", ["MGPBD_NO_EVAL_HV=1", "MGPBD_NO_HALO_OVERLAP=1", "MGPBD_NO_X1_FUSE=1"])
def test_fusions_are_bitwise(monkeypatch, precision, switch):
    """Fusions that move work between kernels without changing any arithmetic give bit-identical frames: the
    evaluation writing the vertex-major data (vs k_mf_refresh), the V-cycle's first step formed by the x/r update
    (vs k_jacobi0), the overlapped halo exchange (one rank: no halo, same path)."""
    sc = scenes.make("block_small")
    outs = []
    for sw in ("", switch):
        for kv in sw.split():
            k, v = kv.split("=")
            monkeypatch.setenv(k, v)
        ctx = mgpbd.Context.from_scene(sc, precision=precision, min_coarse=30)
        ctx.step(sc.dt, ITERS)
        outs.append((ctx.lambdas(), ctx.positions()))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1]), switch
