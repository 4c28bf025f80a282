"""Seeded synthetic workloads for the five BASELINE.json configurations.

This module only BUILDS inputs (A0, Bl, Br, Q, E and the parameter grid V). It holds none
of the method's arithmetic: no Lyapunov solve, no eigendecomposition of A0, no Cauchy
matrix. Both the CPU oracle (oracle/) and the CUDA path (paper_2312_08201_b200/) consume
what it returns, and neither is imported here.

Paper passages the constructions follow (PAPER.md = /root/reference/PAPER.md, read at
authoring time only; nothing reads it at run time):

* Vibrational systems, §3.1: M x'' + C(v) x' + K x = 0 with C(v) = C_int + B D(v) B^T
  (eqs. MDK, Cext); modal linearisation eq. (MatrixA), PAPER.md:816-823:
  A(v) = [[0, Omega], [-Omega, -Phi^T C(v) Phi]], Phi from eq. (MatrixPhi)
  (Phi^T K Phi = Omega^2, Phi^T M Phi = I, omega ascending).  BASELINE fixes the internal
  damping as Phi^T C_int Phi = 2 alpha Omega (reading R2), so
  A0 = [[0, Omega], [-Omega, -2 alpha Omega]], Bl = Br = [0; Phi^T e_p] (R7).
* Multi-agent systems, §3.2 (eqs. MASsystem/protocol) as concretised by
  BASELINE config 3: A0 = I_N (x) S - 0.5 (L_G (x) I_d).
* The parameter sets are tensor grids (BASELINE): numpy.geomspace / numpy.linspace with
  inclusive endpoints, Cartesian product in itertools.product order (last parameter
  fastest), reading R10.

Every config is a pure function of (name, seed); the default seeds are c1->1 ... c5->5.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

__all__ = ["Workload", "make", "CONFIG_NAMES", "grid", "chain", "multi_agent", "random_stable", "rank_grid"]

CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")


@dataclass
class Workload:
    """One problem instance: A(v) = A0 - Bl diag(v) Br^T, Q, E and a batch V of v's."""

    name: str
    A0: np.ndarray  # n x n float64
    Bl: np.ndarray  # n x k
    Br: np.ndarray  # n x k
    Q: np.ndarray  # n x n symmetric
    E: np.ndarray  # n x n symmetric
    V: np.ndarray  # nv x k
    grid_shape: tuple = ()
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.A0.shape[0]

    @property
    def k(self) -> int:
        return self.Bl.shape[1]

    @property
    def nv(self) -> int:
        return self.V.shape[0]

    def corner_indices(self) -> list[int]:
        """Flat indices of the 2^k grid corners and the grid centre (parity samples)."""
        shp = self.grid_shape
        idx = []
        for c in itertools.product(*[(0, s - 1) for s in shp]):
            idx.append(int(np.ravel_multi_index(c, shp)))
        idx.append(int(np.ravel_multi_index(tuple(s // 2 for s in shp), shp)))
        return sorted(set(idx))

    def sample_indices(self, count: int, seed: int = 0) -> np.ndarray:
        """Corners + centre + a seeded uniform sample, sorted, at most `count` (>= corners)."""
        base = self.corner_indices()
        rest = np.setdiff1d(np.arange(self.nv), base)
        rng = np.random.default_rng(1000 + seed)
        extra = max(0, count - len(base))
        pick = rng.choice(rest, size=min(extra, rest.size), replace=False) if extra else []
        return np.array(sorted(set(base) | set(int(i) for i in pick)), dtype=np.int64)


def grid(lo: float, hi: float, g: int, k: int, log: bool) -> np.ndarray:
    """k-dimensional tensor grid, g points per axis, last parameter fastest (reading R10)."""
    axis = np.geomspace(lo, hi, g) if log else np.linspace(lo, hi, g)
    return np.array(list(itertools.product(axis, repeat=k)), dtype=np.float64)


def chain(m: int, kappa: float, alpha: float, positions, masses=None, modes_in_E: int = 10):
    """Modal phase-space form of a fixed-fixed mass-spring chain.

    K = kappa * tridiag(-1, 2, -1); M = diag(masses) (unit if None).
    Returns A0, Bl=Br, Q=I, E=selector of the `modes_in_E` lowest modes in both blocks.
    """
    K = kappa * (2.0 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1))
    M = np.eye(m) if masses is None else np.diag(np.asarray(masses, dtype=np.float64))
    w2, Phi = scipy.linalg.eigh(K, M)  # ascending, Phi^T M Phi = I  (eq. MatrixPhi)
    omega = np.sqrt(w2)
    Om = np.diag(omega)
    n = 2 * m
    A0 = np.zeros((n, n))
    A0[:m, m:] = Om
    A0[m:, :m] = -Om
    A0[m:, m:] = -2.0 * alpha * Om
    k = len(positions)
    B = np.zeros((n, k))
    for t, p in enumerate(positions):  # 1-based mass index (reading R8)
        B[m:, t] = Phi[p - 1, :]  # Phi^T e_p
    Q = np.eye(n)
    sel = np.zeros(n)
    sel[:modes_in_E] = 1.0
    sel[m:m + modes_in_E] = 1.0
    E = np.diag(sel)
    return A0, B.copy(), B.copy(), Q, E, {"omega_min": float(omega[0]), "omega_max": float(omega[-1])}


def _connected_er(N: int, p: float, rng) -> tuple[np.ndarray, int]:
    """Erdos-Renyi G(N, p) adjacency, resampled until connected (reading R12)."""
    attempts = 0
    while True:
        attempts += 1
        U = rng.random((N, N)) < p
        Adj = np.triu(U, 1)
        Adj = (Adj | Adj.T).astype(np.float64)
        # connectivity by BFS (no spectral arithmetic needed)
        seen = np.zeros(N, bool)
        seen[0] = True
        frontier = [0]
        while frontier:
            nxt = []
            for i in frontier:
                for j in np.nonzero(Adj[i])[0]:
                    if not seen[j]:
                        seen[j] = True
                        nxt.append(j)
            frontier = nxt
        if seen.all():
            return Adj, attempts


def multi_agent(N: int, d: int, p: float, k: int, rng):
    """BASELINE config 3: A0 = I_N (x) S - 0.5 (L_G (x) I_d), Bl = Br = (e_i - e_j) (x) e_1."""
    W = np.triu(rng.standard_normal((d, d)), 1)
    S = -0.5 * np.eye(d) + (W - W.T)  # reading R11
    Adj, attempts = _connected_er(N, p, rng)
    LG = np.diag(Adj.sum(1)) - Adj
    A0 = np.kron(np.eye(N), S) - 0.5 * np.kron(LG, np.eye(d))
    non_edges = [(i, j) for i in range(N) for j in range(i + 1, N) if Adj[i, j] == 0]
    pick = rng.choice(len(non_edges), size=k, replace=False)  # reading R13
    e1 = np.zeros(d)
    e1[0] = 1.0
    n = N * d
    B = np.zeros((n, k))
    for t, ix in enumerate(sorted(int(x) for x in pick)):
        i, j = non_edges[ix]
        eij = np.zeros(N)
        eij[i], eij[j] = 1.0, -1.0
        B[:, t] = np.kron(eij, e1)
    Q = np.eye(n)
    E = np.kron(np.eye(N) - np.ones((N, N)) / N, np.outer(e1, e1))
    meta = {"er_attempts": attempts, "edges": int(Adj.sum() // 2),
            "new_edges": [non_edges[int(x)] for x in sorted(int(x) for x in pick)]}
    return A0, B.copy(), B.copy(), Q, E, meta


def random_stable(n: int, k: int, rng, normal: bool = False, same_b: bool = False,
                  shift: float = 0.5):
    """Small random test instance: non-normal A0 with spectrum in Re < -shift/2 (tests only)."""
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    if normal:
        W = np.triu(G, 1)
        A0 = (W - W.T) - shift * np.eye(n)
    else:
        # shift by the spectral abscissa of the symmetric part -> Hurwitz with margin
        a = np.linalg.eigvalsh(0.5 * (G + G.T)).max()
        A0 = G - (a + shift) * np.eye(n)
    Bl = rng.standard_normal((n, k)) / np.sqrt(n)
    Br = Bl.copy() if same_b else rng.standard_normal((n, k)) / np.sqrt(n)
    R = rng.standard_normal((n, n))
    Q = R @ R.T / n + 0.1 * np.eye(n)
    F = rng.standard_normal((n, max(1, n // 3)))
    E = F @ F.T / n
    return A0, Bl, Br, Q, E


def make(name: str, seed: int | None = None) -> Workload:
    """Build BASELINE config `name` (c1..c5) with its default seed (c_i -> i) or `seed`."""
    if name not in CONFIG_NAMES:
        raise ValueError(f"unknown config {name!r}")
    s = int(name[1]) if seed is None else seed
    rng = np.random.default_rng(s)
    if name == "c1":
        A0, Bl, Br, Q, E, meta = chain(50, 100.0, 0.02, [10, 35], modes_in_E=10)
        gspec = (0.1, 100.0, 16, 2, True)
        V, shp = grid(*gspec[:4], log=gspec[4]), (16, 16)
        meta["positions"] = [10, 35]
    elif name == "c2":
        pos = sorted(int(x) + 1 for x in rng.choice(400, 2, replace=False))
        A0, Bl, Br, Q, E, meta = chain(400, 500.0, 0.01, pos, modes_in_E=40)
        gspec = (0.01, 1000.0, 64, 2, True)
        V, shp = grid(*gspec[:4], log=gspec[4]), (64, 64)
        meta["positions"] = pos
    elif name == "c3":
        A0, Bl, Br, Q, E, meta = multi_agent(200, 4, 0.03, 3, rng)
        gspec = (0.05, 5.0, 16, 3, False)
        V, shp = grid(*gspec[:4], log=gspec[4]), (16, 16, 16)
    elif name == "c4":
        masses = rng.uniform(1.0, 3.0, 1000)
        pos = sorted(int(x) + 1 for x in rng.choice(1000, 3, replace=False))
        A0, Bl, Br, Q, E, meta = chain(1000, 1000.0, 0.02, pos, masses=masses, modes_in_E=50)
        gspec = (0.1, 500.0, 20, 3, True)
        V, shp = grid(*gspec[:4], log=gspec[4]), (20, 20, 20)
        meta["positions"] = pos
    else:  # c5
        pos = sorted(int(x) + 1 for x in rng.choice(2000, 4, replace=False))
        A0, Bl, Br, Q, E, meta = chain(2000, 2000.0, 0.005, pos, modes_in_E=100)
        gspec = (0.1, 1000.0, 8, 4, True)
        V, shp = grid(*gspec[:4], log=gspec[4]), (8, 8, 8, 8)
        meta["positions"] = pos
    meta["seed"] = s
    meta["grid_spec"] = gspec  # (lo, hi, points per axis, k, log-spaced)
    return Workload(name, A0, Bl, Br, Q, E, V, shp, meta)


def rank_grid(W: Workload, rank: int, world: int) -> np.ndarray:
    """Weak-scaling grid of one rank: the configuration's grid with axis 0 refined world-fold and
    interleaved (rank r takes refined points r, r + world, ...).  Same size and value distribution
    as W.V on every rank; world = 1 returns W.V exactly."""
    lo, hi, g, k, log = W.meta["grid_spec"]
    if world == 1:
        return W.V
    fine = np.geomspace(lo, hi, g * world) if log else np.linspace(lo, hi, g * world)
    axis0 = fine[rank::world]
    base = np.geomspace(lo, hi, g) if log else np.linspace(lo, hi, g)
    return np.array(list(itertools.product(axis0, *([base] * (k - 1)))), dtype=np.float64)
