"""Seeded synthetic workloads for BASELINE.json's configs (own generator; the
reference's datasets.cpp generators do not match BASELINE's mixture).

G(N, D, K, sigma, seed): K centres c_j ~ N(0, I_D), L2-normalised; each point
x = normalise(s * (c_j + sigma * eps)), j ~ U{0..K-1}, eps ~ N(0, I_D), where s
is the optional per-coordinate anisotropy (config 3: one s ~ U[0.8, 1.2]^D per
dataset, applied before normalisation).  Queries come from the same mixture in a
separate RNG stream.  numpy PCG64 streams: centres/scale `seed`, base `seed+1`,
queries `seed+2`.

sigma_mode "literal" reads sigma per coordinate (noise norm ~ sigma*sqrt(D),
the BASELINE wording, near-structureless); "norm" uses sigma/sqrt(D) per
coordinate (noise norm ~ sigma, clustered) — reported separately.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dim: int
    centers: int
    sigma: float
    m: int            # R = 2m
    ef_c: int         # L
    alpha: float = 1.2
    nq: int = 10_000
    k: int = 10
    efs: tuple = (64,)
    aniso: bool = False


CONFIGS = {
    1: Config("cfg1", 100_000, 384, 1000, 0.35, 16, 64, efs=(64,)),
    2: Config("cfg2", 1_000_000, 768, 4096, 0.3, 32, 128, efs=(16, 32, 64, 128, 256)),
    3: Config("cfg3", 1_000_000, 1536, 8192, 0.25, 32, 128, efs=(64,), aniso=True),
    4: Config("cfg4", 1_000_000, 3072, 4096, 0.3, 32, 128, efs=(64, 128)),
}


def _normalise(x: np.ndarray) -> np.ndarray:
    nrm = np.sqrt(np.einsum("ij,ij->i", x, x, dtype=np.float64)).astype(np.float32)
    nrm[nrm == 0] = 1.0
    x /= nrm[:, None]
    return x


def mixture(n, dim, centers, sigma, seed=42, nq=0, aniso=False, sigma_mode="literal",
            chunk=65536):
    """-> (base[n,dim] f32 unit rows, queries[nq,dim] f32 unit rows)."""
    rc = np.random.Generator(np.random.PCG64(seed))
    cen = rc.standard_normal((centers, dim), dtype=np.float32)
    cen = _normalise(cen)
    scale = rc.uniform(0.8, 1.2, dim).astype(np.float32) if aniso else None
    s = np.float32(sigma if sigma_mode == "literal" else sigma / np.sqrt(dim))

    def draw(count, rng):
        out = np.empty((count, dim), np.float32)
        for r0 in range(0, count, chunk):
            r1 = min(count, r0 + chunk)
            j = rng.integers(0, centers, r1 - r0)
            x = rng.standard_normal((r1 - r0, dim), dtype=np.float32)
            x *= s
            x += cen[j]
            if scale is not None:
                x *= scale
            out[r0:r1] = _normalise(x)
        return out

    base = draw(n, np.random.Generator(np.random.PCG64(seed + 1)))
    queries = draw(nq, np.random.Generator(np.random.PCG64(seed + 2))) if nq else np.empty(
        (0, dim), np.float32)
    return base, queries


def config_data(cfg: Config, n=None, nq=None, sigma_mode="literal", seed=42):
    return mixture(n or cfg.n, cfg.dim, cfg.centers, cfg.sigma, seed=seed,
                   nq=cfg.nq if nq is None else nq, aniso=cfg.aniso, sigma_mode=sigma_mode)
