"""The BASELINE.json configurations and their seeded synthetic inputs.

BASELINE.json lists five configs (the reference publishes no GPU numbers and
its own tests never use these generators).  Inputs follow
DESIGN.md §3: A generated on the device (bit-identical to the oracle's host
generator), b / X0 on the host; X0[:, 0] = 0 and X0[:, j >= 1] ~ U[-1, 1]
because x0 = 0 for every agent makes rank(D0) = 1 and ccg_solve returns
rank-collapse at k = 0 (solvers.hpp:83-85).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .solver import GpuContext, SolveOptions, gen_reference_rhs_starts, gen_rhs, gen_starts


@dataclass(frozen=True)
class Config:
    idx: int
    n: int
    p: int
    matrix: str          # "diagdom" | "householder"
    rhs: str             # "uniform" | "normal"
    reflectors: int = 0
    kappa: float = 1.0
    rel_tol: float = 0.0  # tol = rel_tol * ||b||_2 (0 => fixed iterations)
    fixed_iters: int = -1
    seed: int = 0

    @property
    def name(self) -> str:
        return f"cfg{self.idx}_n{self.n}_p{self.p}_{self.matrix}"


CONFIGS = {
    0: Config(0, 1000, 3, "diagdom", "uniform", rel_tol=1e-10, seed=12040),
    1: Config(1, 4096, 4, "householder", "normal", reflectors=8, kappa=1e4, rel_tol=1e-10, seed=12041),
    2: Config(2, 16384, 8, "diagdom", "uniform", fixed_iters=200, seed=12042),
    3: Config(3, 65536, 16, "householder", "normal", reflectors=16, kappa=1e6, fixed_iters=100, seed=12043),
    4: Config(4, 131072, 32, "diagdom", "uniform", fixed_iters=50, seed=12044),
}


def seq_norm(b: np.ndarray) -> float:
    """sqrt(dot(b, b)) accumulated in ascending order (kernels.hpp:20-26)."""
    sq = np.asarray(b, dtype=np.float64) ** 2
    return float(np.sqrt(np.cumsum(sq)[-1])) if len(sq) else 0.0


def solve_options(cfg: Config, b: np.ndarray) -> SolveOptions:
    if cfg.fixed_iters >= 0:
        return SolveOptions(tol=0.0, max_iters=cfg.fixed_iters)
    return SolveOptions(tol=cfg.rel_tol * seq_norm(b), max_iters=-1)


def host_inputs(cfg: Config, n: int | None = None, p: int | None = None):
    n = n or cfg.n
    p = p or cfg.p
    b = gen_rhs(n, cfg.rhs, cfg.seed)
    X0 = gen_starts(n, p, cfg.seed)
    return b, X0


def make_problem_on_device(ctx: GpuContext, cfg: Config):
    """Generate A on ctx's device and return (b, X0, opts) for cfg."""
    ctx.gen_A(cfg.matrix, cfg.seed, cfg.reflectors, cfg.kappa)
    b, X0 = host_inputs(cfg, ctx.n, ctx.p)
    return b, X0, solve_options(cfg, b)


def make_reference_problem_on_device(ctx: GpuContext, cond: float, seed: int):
    """The reference's make_problem<double>(ProblemSpec{n, p, cond, seed})
    (problem.hpp:219-230) with A generated on ctx's device: A = random_spd(n,
    cond, seed) bit for bit, b / X0 = random_rhs_and_starts (host).  Returns
    (b, X0) for ccg_solve's default options."""
    ctx.gen_A("random_spd", seed, 0, cond)
    return gen_reference_rhs_starts(ctx.n, ctx.p, seed)
