"""Synthetic low-rank + sparse inputs generated directly in HBM.

The reference generator (spcp synth.py:13-57) builds X = A B^T + S + noise on
the host with numpy; at 20000 x 20000 that is 3.2 GB per float64 array and
the 200000 x 20000 shape (32 GB) cannot be built on the host at all
(SURVEY §8(d), §8(f) row 3).  This generator keeps the same law:

  * A (m x rank), B (n_total x rank) i.i.d. N(0, 1) from numpy's PCG64 stream
    seeded like the reference (so L_ref = A B^T is the reference's);
  * outliers: each entry is an outlier with probability `sparse_frac`, value
    N(0, 1) (Bernoulli instead of an exact count);
  * Gaussian noise with the variance that makes E|noise|^2 / E|X|^2 =
    noise_rel^2 (instead of the exact per-draw ratio);

with the outliers/noise drawn by torch's counter-based CUDA Philox stream
keyed by (seed, first column, row chunk), so each column shard of a sharded
problem generates its own columns without communication.  Input synthesis is
not part of the measured path.
"""

import math

import numpy as np

__all__ = ["gen_low_rank_plus_sparse", "gen_mask", "gen_low_rank_plus_sparse_device",
           "factor_draw"]


def factor_draw(m, n_total, rank, seed):
    """A (m x rank), B (n_total x rank) exactly as synth.py:31-33 draws them."""
    gen = np.random.default_rng(seed)
    a = gen.standard_normal((m, rank))
    b = gen.standard_normal((n_total, rank))
    return a, b


def gen_low_rank_plus_sparse(m, n, rank, sparse_frac, noise_rel, seed=0):
    """(x, l_ref, s_ref) on the host, byte-identical to synth.py:13-57 for a
    seed: the same PCG64 draws in the same order (A, B, outlier positions and
    values, noise field) and the exact noise ratio, from the positive root of
    |a z|^2 = rho^2 |clean + a z|^2.  Feeds the CLI's `synth` command; the
    benchmark shapes use the device generator below."""
    m, n, rank = int(m), int(n), int(rank)
    if rank < 0 or rank > min(m, n):
        raise ValueError(f"rank={rank} out of range [0, {min(m, n)}]")
    if not 0.0 <= sparse_frac <= 1.0:
        raise ValueError(f"sparse_frac={sparse_frac} out of range [0, 1]")
    if not 0.0 <= noise_rel < 1.0:
        raise ValueError(f"noise_rel={noise_rel} out of range [0, 1)")
    gen = np.random.default_rng(seed)
    a = gen.standard_normal((m, rank))
    b = gen.standard_normal((n, rank))
    l_ref = a @ b.T
    s_ref = np.zeros((m, n))
    count = int(round(sparse_frac * m * n))
    if count:
        where = gen.choice(m * n, size=count, replace=False)
        s_ref.reshape(-1)[where] = gen.standard_normal(count)
    clean = l_ref + s_ref
    if noise_rel == 0.0:
        return clean.copy(), l_ref, s_ref
    noise = gen.standard_normal((m, n))
    r2 = noise_rel * noise_rel
    nn = float(np.sum(noise * noise))
    nc = float(np.sum(clean * noise))
    cc = float(np.sum(clean * clean))
    qa, qb, qc = nn * (1.0 - r2), -2.0 * r2 * nc, -r2 * cc
    scale = (-qb + np.sqrt(qb * qb - 4.0 * qa * qc)) / (2.0 * qa)
    return clean + scale * noise, l_ref, s_ref


def gen_mask(m, n, observe_frac, seed=0):
    """Exactly round(observe_frac m n) observed positions, uniform without
    replacement (synth.py:60-73)."""
    m, n = int(m), int(n)
    if not 0.0 < observe_frac <= 1.0:
        raise ValueError(f"observe_frac={observe_frac} out of range (0, 1]")
    hits = np.random.default_rng(seed).choice(m * n, size=int(round(observe_frac * m * n)),
                                              replace=False)
    mask = np.zeros(m * n, dtype=bool)
    mask[hits] = True
    return mask.reshape(m, n)


def gen_low_rank_plus_sparse_device(m, n, rank, sparse_frac, noise_rel, seed=0, col0=0,
                                    n_total=None, dtype="float32", chunk_rows=2048,
                                    device=None):
    """X[:, col0:col0+n] of the synthetic problem as a CUDA tensor (m x n)."""
    import torch

    n_total = n if n_total is None else n_total
    dev = device or torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if dtype == "float32" else torch.float64
    a, b = factor_draw(m, n_total, rank, seed)
    a_d = torch.from_numpy(a).to(dev)
    b_d = torch.from_numpy(np.ascontiguousarray(b[col0:col0 + n])).to(dev)
    c = rank + sparse_frac
    sigma = noise_rel * math.sqrt(c / (1.0 - noise_rel * noise_rel)) if noise_rel > 0 else 0.0
    out = torch.empty((m, n), dtype=tdt, device=dev)
    gen = torch.Generator(device=dev)
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        gen.manual_seed(int(seed) * 1_000_003 + int(col0) * 7919 + r0)
        blk = a_d[r0:r1] @ b_d.T
        if sparse_frac > 0:
            hit = torch.rand((r1 - r0, n), generator=gen, device=dev, dtype=torch.float64)
            vals = torch.randn((r1 - r0, n), generator=gen, device=dev, dtype=torch.float64)
            blk += torch.where(hit < sparse_frac, vals, torch.zeros_like(vals))
            del hit, vals
        if sigma > 0:
            blk += sigma * torch.randn((r1 - r0, n), generator=gen, device=dev,
                                       dtype=torch.float64)
        out[r0:r1] = blk.to(tdt)
        del blk
    return out
