"""The five BASELINE.json configs (C1-C5) and reduced-size variants.

Each config fixes the mesh generator, k, the K field, the preconditioner(s),
the GMRES restart m and rtol (readings R12-R18).
The reduced variants keep the structure (K-field shape, pairing, jitter) at
sizes the oracle finishes in seconds; they are parity cases, not bench lines.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mesh as _mesh
from .assemble import build_system

BLOCK_SCHUR = 1
BLOCK_REG = 2


def lognormal_block_K(n: int, block: int, seed: int, lo=-4.0, hi=0.0):
    """C3: scalar K constant on block^3-cube blocks, 10^U(lo, hi), seeded."""
    nb = n // block
    rng = np.random.Generator(np.random.PCG64(seed))
    kb = 10.0 ** rng.uniform(lo, hi, size=nb ** 3)
    idx = np.arange(n ** 3)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    b = (i // block) + nb * ((j // block) + nb * (k // block))
    return np.repeat(kb[b][:, None], 3, axis=1)


def checker_aniso_K(n: int, block: int, seed: int):
    """C5: K = diag(1, 1, 1e-2) * c, c = 1e-3 on odd checkerboard blocks
    (phase from the seed), else 1 (reading R14)."""
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    phase = int(rng.integers(0, 2))
    idx = np.arange(n ** 3)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    odd = ((i // block) + (j // block) + (k // block) + phase) % 2 == 1
    c = np.where(odd, 1e-3, 1.0)
    return np.stack([c, c, 1e-2 * c], axis=1)


@dataclass
class Config:
    name: str
    kind: str          # cube | kuhn | pairs
    n: int
    k: int
    precs: tuple
    restart: int
    rtol: float = 1e-10
    block: int = 0     # K block size (cubes) / pairing block (pairs)
    seed: int = 0
    describe: str = ""
    paper: bool = False   # the paper's own BDM-type space (pressure P_{k-1}), SURVEY.md N3

    def make_mesh(self):
        if self.kind == "cube":
            K = lognormal_block_K(self.n, self.block, self.seed) if self.block else None
            return _mesh.cube_mesh(self.n, K)
        if self.kind == "kuhn":
            return _mesh.kuhn_mesh(self.n, seed=self.seed, jitter=0.2)
        if self.kind == "pairs":
            Kc = checker_aniso_K(self.n, self.block, self.seed)
            return _mesh.pair_mesh(self.n, seed=self.seed, block=self.block, Kcell=Kc)
        raise ValueError(self.kind)

    def build(self, keep_local=False):
        return build_system(self.make_mesh(), self.k, keep_local=keep_local, paper_mode=self.paper)


CONFIGS = {
    "C1": Config("C1", "cube", 8, 0, (BLOCK_SCHUR,), 30,
                 describe="8^3 cubes, k=0, K=I, Block-Schur, GMRES(30)"),
    "C2": Config("C2", "kuhn", 16, 1, (BLOCK_SCHUR, BLOCK_REG), 30, seed=2,
                 describe="16^3x6 Kuhn tets +-0.2h, k=1, K=I, both preconditioners"),
    "C3": Config("C3", "cube", 128, 0, (BLOCK_SCHUR,), 50, block=8, seed=3,
                 describe="128^3 cubes, k=0, K log-uniform [1e-4,1] on 8^3 blocks, Block-Schur, GMRES(50)"),
    "C4": Config("C4", "cube", 48, 2, (BLOCK_SCHUR, BLOCK_REG), 50,
                 describe="48^3 cubes, k=2, K=I, both preconditioners, GMRES(50)"),
    "C5": Config("C5", "pairs", 96, 1, (BLOCK_REG,), 50, block=12, seed=5,
                 describe="96^3 cubes, ~50% pairs, k=1, K=diag(1,1,1e-2)*checker{1,1e-3}, Block-Reg, GMRES(50)"),
    # reduced variants (parity cases)
    "C2s": Config("C2s", "kuhn", 4, 1, (BLOCK_SCHUR, BLOCK_REG), 30, seed=2),
    "C3s": Config("C3s", "cube", 16, 0, (BLOCK_SCHUR,), 50, block=2, seed=3),
    "C4s": Config("C4s", "cube", 6, 2, (BLOCK_SCHUR, BLOCK_REG), 50),
    "C5s": Config("C5s", "pairs", 12, 1, (BLOCK_REG,), 50, block=3, seed=5),
    # C5-type at 6^3 (two K blocks per axis): the size at which the oracle finishes the
    # kind-5 solve (PCG on M + B^T (eps W)^-1 B inside FGMRES, R24) in seconds
    "C5t": Config("C5t", "pairs", 6, 1, (BLOCK_REG,), 50, block=3, seed=5),
    # paper mode (N3): the paper's BDM-type space on cube grids, K = I (its Tables 1 and 4 use Cube
    # meshes at k = 1, 2), with this build's Dirichlet pressure data (R5)
    "P1s": Config("P1s", "cube", 6, 1, (BLOCK_SCHUR, BLOCK_REG), 50, paper=True,
                  describe="6^3 cubes, paper-mode k=1 (pressure P0)"),
    "P2s": Config("P2s", "cube", 4, 2, (BLOCK_SCHUR, BLOCK_REG), 50, paper=True,
                  describe="4^3 cubes, paper-mode k=2 (pressure P1)"),
}


def paper_cube(n: int, k: int) -> Config:
    """Cube n^3 in paper mode at order k (the meshes of PAPER.md Table 4: n = 8, 16, 20, 24, 28 at k = 2)."""
    return Config(f"paper-cube{n}-k{k}", "cube", n, k, (BLOCK_SCHUR, BLOCK_REG), 50, paper=True)


def eps_for(system) -> float:
    """Block-Reg regularisation eps = 1e-6 * mean diag(M) (BASELINE.json C2)."""
    return 1e-6 * float(system.M.diagonal().mean())


def random_rhs(n: int, seed: int = 7) -> np.ndarray:
    """the benchmark extra -- the same matrices with a
    seeded N(0, 1) right-hand side (seed 7).  With K = I on uniform cubes the sin
    source is nearly an eigenvector (R21) and iteration counts are not
    representative; this RHS is."""
    return np.random.default_rng(seed).standard_normal(n)


def paper_neumann(n: int, k: int):
    """The paper's own boundary value problem on the n^3 cube grid at order k:
    BDM-type space, nu = 1, the polynomial solution of PAPER.md P:898-911, Neumann data on the
    whole boundary and the mean-value multiplier.  Returns (System, NeumannSystem)."""
    from .assemble import neumann_system, paper_exact_u, paper_source
    s = build_system(_mesh.cube_mesh(n), k, source=paper_source, keep_local=True, paper_mode=True)
    return s, neumann_system(s, paper_exact_u)
