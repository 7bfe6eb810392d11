"""Seeded synthetic workloads for BASELINE.json's five configs (SURVEY.md §8 d).

The reference ships no dataset; BASELINE.json describes five synthetic
matrices.  These recipes (numpy PCG64 ``default_rng``, seed = config number,
draws in the order written) are the ones SURVEY.md §8(d) fixes, so every run,
test and fixture sees the same data.  ``t`` may be overridden to draw a
smaller matrix with the same recipe (used by parity tests and the CPU
baseline's bounded sample).

Bench/test infrastructure: not part of the product package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    t: int
    n: int
    b: int
    m: int
    desc: str


CONFIGS = {
    "cfg1": Config("cfg1", 20_000, 24, 4, 4, "iid N(0,1); cols 0-3 cubed, 4-7 exp"),
    "cfg2": Config("cfg2", 1_000_000, 64, 8, 4, "Gaussian copula Z@L, Student-t(5) marginals"),
    "cfg3": Config("cfg3", 2_000_000, 48, 4, 5, "Gamma(2,1) | Laplace(0,1) halves"),
    "cfg4": Config("cfg4", 1_000_000, 36, 3, 6, "3-component Gaussian mixture"),
    "cfg5": Config("cfg5", 4_000_000, 96, 6, 6, "Gaussian copula, Student-t(5), n=96"),
}


def _student_copula(rng: np.random.Generator, t: int, n: int) -> np.ndarray:
    import os
    from concurrent.futures import ThreadPoolExecutor

    from scipy import special

    lower = np.tril(rng.uniform(-0.3, 0.3, (n, n)), -1) + np.eye(n)
    z = rng.standard_normal((t, n))
    y = z @ lower
    s = np.sqrt((lower ** 2).sum(0))
    # sf/isf form: ppf(1.0) = inf would be rejected by the finite check.
    # stats.norm.sf(v) == special.ndtr(-v) and stats.t.isf(q, 5) ==
    # -special.stdtrit(5, q) bit for bit; the ufuncs run chunked on threads.
    q = special.ndtr(-(np.abs(y) / s)).ravel()
    out = np.empty_like(q)
    bounds = np.linspace(0, q.size, 65).astype(np.int64)

    def work(i):
        lo, hi = bounds[i], bounds[i + 1]
        out[lo:hi] = special.stdtrit(5, q[lo:hi])

    with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(64)))
    return np.sign(y) * -out.reshape(y.shape)


def generate(name: str, t: int | None = None, shard: int = 0) -> np.ndarray:
    """The (t x n) float64 matrix of config ``name`` (C-contiguous).

    ``shard`` > 0 draws an independent shard of the same distribution (seed
    offset by 1000 * shard) for weak-scaling runs on several GPUs; shard 0 is
    the canonical recipe."""
    cfg = CONFIGS[name]
    t = cfg.t if t is None else int(t)
    off = 1000 * int(shard)
    if name == "cfg1":
        rng = np.random.default_rng(1 + off)
        z = rng.standard_normal((t, 24))
        x = z.copy()
        x[:, 0:4] = z[:, 0:4] ** 3
        x[:, 4:8] = np.exp(z[:, 4:8])
    elif name == "cfg2":
        x = _student_copula(np.random.default_rng(2 + off), t, 64)
    elif name == "cfg3":
        rng = np.random.default_rng(3 + off)
        x = np.empty((t, 48))
        x[:, :24] = rng.gamma(2.0, 1.0, (t, 24))
        x[:, 24:] = rng.laplace(0.0, 1.0, (t, 24))
    elif name == "cfg4":
        rng = np.random.default_rng(4 + off)
        mu = rng.uniform(-2, 2, (3, 36))
        z = rng.choice(3, size=t, p=[0.5, 0.3, 0.2])
        x = mu[z] + rng.standard_normal((t, 36))
    elif name == "cfg5":
        x = _student_copula(np.random.default_rng(5 + off), t, 96)
    else:
        raise KeyError(name)
    return np.ascontiguousarray(x, dtype=np.float64)


def stored_elements(n: int, k: int, b: int) -> int:
    """S_k: stored elements of an order-k packed tensor (sum of block sizes)."""
    from itertools import combinations_with_replacement
    from math import prod

    nb = -(-n // b)
    if n % b == 0:
        from math import comb

        return b ** k * comb(nb + k - 1, k)
    return sum(prod(min(j * b, n) - (j - 1) * b for j in key)
               for key in combinations_with_replacement(range(1, nb + 1), k))


def moment_flops(t: int, n: int, b: int, m_max: int) -> float:
    """Algorithmic FLOPs of cumulants_upto's moments: sum_k 2 t S_k, k=2..m."""
    return float(sum(2.0 * t * stored_elements(n, k, b) for k in range(2, m_max + 1)))
