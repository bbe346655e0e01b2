"""Seeded synthetic inputs shaped like the paper's scenes (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no constraint evaluation, no assembly, no
AMG): it only builds meshes, masses, pins, compliance and initial states, as described in
DESIGN.md "Input recipe".  Both the CUDA path and the oracle consume its output.

Scenes (Table 1):
  * cloth N:  (N+1)^2 vertices, vertical sheet x in [0,1], y in [0,1]; vertex (i,j) at
    (j/N, 1-i/N, 0); distance constraints on horizontal, vertical and the fixed diagonal
    (i,j)-(i+1,j+1) edges (m = 3N^2 + 2N), ordered by quad row ("distance
    constraints"; edge set reading c16).  Total mass 1 kg, uniform; the two top corners
    pinned (w = 0).  alpha = 1/stiffness (Table 1 cloth stiffness 1e9).  Out-of-plane jitter
    1e-2 * (1/N) * (2U-1) with U from hash stream 5.
  * Kuhn block nx x ny x nz cells of size h: each cell split into 6 tets (one per axis
    permutation), cells in x-major order, conforming, positively oriented.  Density 1000,
    lumped V/4 per incident tet, x = 0 face pinned, alpha = 1/(mu V_tet).
    Initial state: squash along y about the centre, a linear twist about the x axis, then
    jitter 1e-3*h*(2U-1) per coordinate (stream 5); rest positions are unjittered.

The hash below is the splitmix64 finaliser (reading c0); the method's own randomness
(aggregation order, colouring order, bootstrap start, power-method start) is implemented
independently inside the oracle and inside the CUDA library.  Here it only jitters inputs.
"""
from __future__ import annotations

import dataclasses
import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def hash_uniform(seed: int, stream: int, level: int, idx: np.ndarray) -> np.ndarray:
    """U(stream, level, i) = ((key >> 11) + 0.5) * 2^-53, key = mix64(mix64(seed^(stream<<56)^(level<<48)) ^ i)."""
    base = np.uint64((seed ^ (stream << 56) ^ (level << 48)) & 0xFFFFFFFFFFFFFFFF)
    k0 = _mix64(np.array([base], dtype=np.uint64))[0]
    key = _mix64(np.asarray(idx, dtype=np.uint64) ^ k0)
    return ((key >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


@dataclasses.dataclass
class Scene:
    name: str
    kind: int                 # 2 = distance (cloth), 4 = tet ARAP
    verts: np.ndarray         # (m, kind) int32
    rest_pos: np.ndarray      # (n, 3) float64
    pos: np.ndarray           # (n, 3) float64, initial positions
    vel: np.ndarray           # (n, 3) float64
    inv_mass: np.ndarray      # (n,) float64, 0 = pinned
    compliance: np.ndarray    # (m,) float64, alpha (NOT divided by dt^2)
    dt: float
    omega_relax: float
    n_iters: int = 20
    pcg_iters: int = 10

    @property
    def n_verts(self) -> int:
        return int(self.rest_pos.shape[0])

    @property
    def n_cons(self) -> int:
        return int(self.verts.shape[0])


def cloth_edges(N: int) -> np.ndarray:
    """Edges of the triangulated N x N quad grid, ordered by quad row.

    Row i (0..N): horizontal edges (i,j)-(i,j+1); then, for i < N, vertical edges
    (i,j)-(i+1,j) for j = 0..N and diagonals (i,j)-(i+1,j+1) for j = 0..N-1.
    """
    vid = lambda i, j: i * (N + 1) + j  # noqa: E731
    out = []
    j = np.arange(N)
    jj = np.arange(N + 1)
    for i in range(N + 1):
        out.append(np.stack([vid(i, j), vid(i, j + 1)], 1))
        if i < N:
            out.append(np.stack([vid(i, jj), vid(i + 1, jj)], 1))
            out.append(np.stack([vid(i, j), vid(i + 1, j + 1)], 1))
    return np.concatenate(out, 0).astype(np.int32)


def cloth(N: int, dt: float = 3e-3, stiffness: float = 1e9, omega_relax: float = 0.25,
          seed: int = 1, jitter: float = 1e-2, n_iters: int = 10, pcg_iters: int = 10,
          name: str | None = None) -> Scene:
    n = (N + 1) * (N + 1)
    i, j = np.divmod(np.arange(n), N + 1)
    rest = np.stack([j / N, 1.0 - i / N, np.zeros(n)], 1).astype(np.float64)
    pos = rest.copy()
    pos[:, 2] = jitter * (1.0 / N) * (2.0 * hash_uniform(seed, 5, 0, np.arange(n)) - 1.0)
    inv_mass = np.full(n, float(n))           # total mass 1 kg, uniform
    inv_mass[0] = 0.0                         # (0,0)
    inv_mass[N] = 0.0                         # (0,N)
    edges = cloth_edges(N)
    comp = np.full(edges.shape[0], 1.0 / stiffness)
    return Scene(name or f"cloth{N}", 2, edges, rest, pos, np.zeros_like(rest), inv_mass,
                 comp, dt, omega_relax, n_iters, pcg_iters)


_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_tets(nx: int, ny: int, nz: int) -> np.ndarray:
    """Kuhn-6 split of an nx*ny*nz lattice; cells x-major, 6 consecutive tets per cell."""
    def vid(a, b, c):
        return (a * (ny + 1) + b) * (nz + 1) + c
    a, b, c = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    a, b, c = a.ravel(), b.ravel(), c.ravel()
    tets = np.empty((a.size, 6, 4), np.int64)
    for t, p in enumerate(_PERMS):
        cur = [a.copy(), b.copy(), c.copy()]
        vs = [vid(*cur)]
        for ax in p:
            cur[ax] = cur[ax] + 1
            vs.append(vid(*cur))
        v = np.stack(vs, 1)
        # orientation of the unit-cube path is the permutation's parity; odd -> swap v1,v2
        parity = sum(1 for x in range(3) for y in range(x + 1, 3) if p[x] > p[y]) % 2
        if parity == 1:
            v[:, [1, 2]] = v[:, [2, 1]]
        tets[:, t, :] = v
    return tets.reshape(-1, 4).astype(np.int32)


def kuhn_block(nx: int, ny: int, nz: int, h: float, mu: float = 1e9, rho: float = 1000.0,
               dt: float = 3e-3, omega_relax: float = 0.1, squash: float = 0.7,
               twist_deg: float = 45.0, jitter: float = 1e-3, seed: int = 1,
               n_iters: int = 20, pcg_iters: int = 10, name: str | None = None) -> Scene:
    a, b, c = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    rest = np.stack([a.ravel() * h, b.ravel() * h, c.ravel() * h], 1).astype(np.float64)
    n = rest.shape[0]
    tets = kuhn_tets(nx, ny, nz)
    # rest volumes (input preparation: masses and compliance are inputs of the method)
    d = rest[tets[:, 1:]] - rest[tets[:, :1]]
    vol = np.abs(np.linalg.det(d)) / 6.0
    mass = np.zeros(n)
    np.add.at(mass, tets.ravel(), np.repeat(rho * vol / 4.0, 4))
    inv_mass = 1.0 / mass
    inv_mass[rest[:, 0] == 0.0] = 0.0        # x = 0 face pinned
    comp = 1.0 / (mu * vol)
    # initial deformed state: squash along y, linear twist about the x axis, jitter
    yc, zc, L = 0.5 * ny * h, 0.5 * nz * h, nx * h
    y = yc + squash * (rest[:, 1] - yc)
    z = rest[:, 2] - zc
    th = np.deg2rad(twist_deg) * rest[:, 0] / L
    pos = np.stack([rest[:, 0], yc + np.cos(th) * (y - yc) - np.sin(th) * z,
                    zc + np.sin(th) * (y - yc) + np.cos(th) * z], 1)
    u = hash_uniform(seed, 5, 0, np.arange(3 * n)).reshape(n, 3)
    pos = pos + jitter * h * (2.0 * u - 1.0)
    return Scene(name or f"block{nx}x{ny}x{nz}", 4, tets, rest, pos, np.zeros_like(rest),
                 inv_mass, comp, dt, omega_relax, n_iters, pcg_iters)


def make(name: str) -> Scene:
    """Named configurations (BASELINE.json configs; SURVEY.md §8(d) sizing table)."""
    if name == "cloth16":
        return cloth(16, dt=3e-3, n_iters=10, pcg_iters=10, name=name)
    if name == "cloth64":
        return cloth(64, dt=3e-3, n_iters=10, pcg_iters=10, name=name)
    if name == "cloth256":
        return cloth(256, dt=20e-3, n_iters=20, pcg_iters=10, name=name)
    if name == "cloth2048":
        return cloth(2048, dt=3e-3, n_iters=20, pcg_iters=10, name=name)
    if name == "bar_small":      # 4x2x2 cells = 96 tets (single-level hierarchy)
        return kuhn_block(4, 2, 2, 0.05, dt=10e-3, squash=1.0, twist_deg=90.0, n_iters=5,
                          name=name)
    if name == "bar3k":          # 20x5x5 cells = 3000 tets (multi-level)
        return kuhn_block(20, 5, 5, 0.05, dt=10e-3, squash=1.0, twist_deg=90.0, n_iters=5,
                          name=name)
    if name == "block_small":    # 24x12x6 cells = 10,368 tets: the block's deformation at desk size
        return kuhn_block(24, 12, 6, 0.01, dt=3e-3, squash=0.7, twist_deg=45.0 * 24 / 136, n_iters=5,
                          name=name)
    if name == "bar50k":         # 60x12x12 cells = 51,840 tets, 5:1:1 (bar twist PAPER.md:330)
        return kuhn_block(60, 12, 12, 1.0 / 60.0, dt=10e-3, squash=1.0, twist_deg=90.0,
                          n_iters=20, name=name)
    if name == "block1.67M":     # 136x64x32 cells = 1,671,168 tets (muscle-human size)
        return kuhn_block(136, 64, 32, 0.01, dt=3e-3, squash=0.7, twist_deg=45.0,
                          n_iters=20, name=name)
    if name.startswith("blockslab"):  # blockslabK: the first K x-slabs of the 1.67M block (CPU samples)
        k = int(name[len("blockslab"):])
        return kuhn_block(k, 64, 32, 0.01, dt=3e-3, squash=0.7, twist_deg=45.0,
                          n_iters=20, name=name)
    raise KeyError(name)
