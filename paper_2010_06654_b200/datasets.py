"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE names no public dataset (the paper's UCI/other datasets are absent);
these generators follow the configs' stated distributions exactly
(SURVEY.md §8d).  Data are float32, rows in random order.  Initial centroids
come from init_random(RunContext(seed=SEED_INIT), x, k), i.e. the reference's
own seeding (core.py:182-189).

Generation is chunked (fixed 1M-row chunks, each with its own PCG64 stream
keyed on (seed, chunk)), so a config can also be produced at a reduced row
count for CPU-oracle parity with the same centres/weights.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import RunContext, init_random

CHUNK = 1 << 20


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    k: int
    t_max: int
    seed_data: int
    seed_init: int
    note: str


CONFIGS = {
    "cfg1": Config("cfg1", 100_000, 16, 100, 50, 1001, 2001,
                   "100 isotropic Gaussians, centres U[-10,10]^16, sigma 1, equal weights"),
    "cfg2": Config("cfg2", 1_000_000, 2, 1000, 100, 1002, 2002,
                   "1000 Gaussians, centres U[0,1000]^2, sigma U[1,10], Dirichlet(1) weights"),
    "cfg3": Config("cfg3", 2_000_000, 128, 1024, 30, 1003, 2003,
                   "1024 Gaussians, unit-norm random centres x4, sigma 1, equal weights"),
    "cfg4": Config("cfg4", 500_000, 784, 256, 30, 1004, 2004,
                   "clip(centre + N(0,0.15)), 256 sparse U[0,1] centres (20% nonzero)"),
    "cfg5": Config("cfg5", 50_000_000, 32, 4096, 20, 1005, 2005,
                   "4096 Gaussians, centres U[-50,50]^32, sigma U[0.5,3], Zipf(1.1) weights"),
}


def _mixture(cfg: Config):
    """Centres [k,d], per-cluster sigma [k], weights [k] (None = equal split)."""
    rng = np.random.default_rng(cfg.seed_data)
    k, d = cfg.k, cfg.d
    if cfg.name == "cfg1":
        return rng.uniform(-10.0, 10.0, size=(k, d)), np.full(k, 1.0), None
    if cfg.name == "cfg2":
        c = rng.uniform(0.0, 1000.0, size=(k, d))
        s = rng.uniform(1.0, 10.0, size=k)
        w = rng.dirichlet(np.ones(k))
        return c, s, w
    if cfg.name == "cfg3":
        g = rng.standard_normal(size=(k, d))
        c = 4.0 * g / np.linalg.norm(g, axis=1, keepdims=True)
        return c, np.full(k, 1.0), None
    if cfg.name == "cfg4":
        nz = rng.random(size=(k, d)) < 0.2
        c = np.where(nz, rng.random(size=(k, d)), 0.0)
        return c, np.full(k, 0.15), None
    if cfg.name == "cfg5":
        c = rng.uniform(-50.0, 50.0, size=(k, d))
        s = rng.uniform(0.5, 3.0, size=k)
        r = np.arange(1, k + 1, dtype=np.float64)
        w = r ** -1.1
        return c, s, w / w.sum()
    raise KeyError(cfg.name)


def generate(name: str, n: int | None = None, *, with_labels: bool = False):
    """Float32 points of config ``name`` (optionally only the first ``n`` rows
    of the same stream).  Returns x, or (x, true_labels)."""
    cfg = CONFIGS[name]
    n_full = cfg.n
    n = n_full if n is None else int(n)
    centres, sigma, weights = _mixture(cfg)
    k, d = cfg.k, cfg.d
    x = np.empty((n, d), dtype=np.float32)
    lab = np.empty(n, dtype=np.int32) if with_labels else None
    if weights is None:
        # equal weights: exact round-robin split of the FULL row count, then one
        # global permutation (so a prefix is an iid-looking sample)
        perm_rng = np.random.default_rng([cfg.seed_data, 0xFFFF])
        order = perm_rng.permutation(n_full)[:n]
        labels_all = (order % k).astype(np.int64)
    for c0 in range(0, n, CHUNK):
        c1 = min(n, c0 + CHUNK)
        rng = np.random.default_rng([cfg.seed_data, c0 // CHUNK])
        if weights is None:
            lb = labels_all[c0:c1]
        else:
            lb = rng.choice(k, size=c1 - c0, p=weights)
        noise = rng.standard_normal(size=(c1 - c0, d), dtype=np.float32)
        blk = centres[lb].astype(np.float32) + noise * sigma[lb, None].astype(np.float32)
        if name == "cfg4":
            np.clip(blk, 0.0, 1.0, out=blk)
        x[c0:c1] = blk
        if with_labels:
            lab[c0:c1] = lb
    return (x, lab) if with_labels else x


def generate_rows(name: str, r0: int, r1: int) -> np.ndarray:
    """Rows r0..r1-1 of the full config ``name`` -- bit-identical to
    generate(name)[r0:r1] -- generating only the 1M-row chunks that overlap
    the range (one rank's shard; no rank materializes the whole matrix)."""
    cfg = CONFIGS[name]
    r0, r1 = max(0, int(r0)), min(cfg.n, int(r1))
    centres, sigma, weights = _mixture(cfg)
    k, d = cfg.k, cfg.d
    out = np.empty((max(0, r1 - r0), d), dtype=np.float32)
    if r1 <= r0:
        return out
    if weights is None:
        perm_rng = np.random.default_rng([cfg.seed_data, 0xFFFF])
        order = perm_rng.permutation(cfg.n)
    for c0 in range((r0 // CHUNK) * CHUNK, r1, CHUNK):
        c1 = min(cfg.n, c0 + CHUNK)
        rng = np.random.default_rng([cfg.seed_data, c0 // CHUNK])
        if weights is None:
            lb = (order[c0:c1] % k).astype(np.int64)
        else:
            lb = rng.choice(k, size=c1 - c0, p=weights)
        noise = rng.standard_normal(size=(c1 - c0, d), dtype=np.float32)
        blk = centres[lb].astype(np.float32) + noise * sigma[lb, None].astype(np.float32)
        if name == "cfg4":
            np.clip(blk, 0.0, 1.0, out=blk)
        a0, a1 = max(c0, r0), min(c1, r1)
        out[a0 - r0:a1 - r0] = blk[a0 - c0:a1 - c0]
    return out


def init_from_rows(name: str, seed: int | None = None) -> np.ndarray:
    """init_random(RunContext(seed), generate(name), k) without the full
    matrix: the same rng.choice draw (core.py:182-189), then only the chunks
    holding the chosen rows."""
    cfg = CONFIGS[name]
    ctx = RunContext(seed=cfg.seed_init if seed is None else seed)
    idx = ctx.rng.choice(cfg.n, size=cfg.k, replace=False)
    out = np.empty((cfg.k, cfg.d), dtype=np.float64)
    chunks = sorted(set(int(i) // CHUNK for i in idx))
    for ch in chunks:
        blk = generate_rows(name, ch * CHUNK, min(cfg.n, (ch + 1) * CHUNK))
        sel = np.nonzero(idx // CHUNK == ch)[0]
        out[sel] = blk[idx[sel] - ch * CHUNK]
    return out


def initial_centroids(name: str, x: np.ndarray, seed: int | None = None) -> np.ndarray:
    """The reference's random init on these points (fp64, [k, d])."""
    cfg = CONFIGS[name]
    return init_random(RunContext(seed=cfg.seed_init if seed is None else seed), x, cfg.k)
