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

__all__ = ["gen_low_rank_plus_sparse", "gen_mask", "gen_low_rank_plus_sparse_device", "gen_video_device",
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


GEN_COL_BLOCK = 512  # counter-stream granularity: any sharding on these boundaries agrees


def gen_low_rank_plus_sparse_device(m, n, rank, sparse_frac, noise_rel, seed=0, col0=0,
                                    n_total=None, dtype="float32", chunk_rows=8192,
                                    device=None):
    """X[:, col0:col0+n] of the synthetic problem as a CUDA tensor (m x n).

    The outlier/noise draws are keyed by (seed, global column block of
    GEN_COL_BLOCK columns, row chunk), never by the shard: a column shard is
    bit-identical to the same columns of the unsharded matrix, so the 1-, 2-,
    4- and 8-GPU runs of a strong-scaling benchmark solve the same problem."""
    import torch

    n_total = n if n_total is None else n_total
    dev = device or torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if dtype == "float32" else torch.float64
    a, b = factor_draw(m, n_total, rank, seed)
    a_d = torch.from_numpy(a).to(dev)
    c = rank + sparse_frac
    sigma = noise_rel * math.sqrt(c / (1.0 - noise_rel * noise_rel)) if noise_rel > 0 else 0.0
    out = torch.empty((m, n), dtype=tdt, device=dev)
    gen = torch.Generator(device=dev)
    cb = GEN_COL_BLOCK
    for blk0 in range((col0 // cb) * cb, col0 + n, cb):
        blk1 = min(blk0 + cb, n_total)
        lo, hi = max(blk0, col0), min(blk1, col0 + n)  # overlap with this shard
        b_d = torch.from_numpy(np.ascontiguousarray(b[blk0:blk1])).to(dev)
        for r0 in range(0, m, chunk_rows):
            r1 = min(m, r0 + chunk_rows)
            gen.manual_seed(int(seed) * 1_000_003 + (blk0 // cb) * 7919 + r0)
            tile = a_d[r0:r1] @ b_d.T
            shape = (r1 - r0, blk1 - blk0)
            if sparse_frac > 0:
                hit = torch.rand(shape, generator=gen, device=dev, dtype=torch.float64)
                vals = torch.randn(shape, generator=gen, device=dev, dtype=torch.float64)
                tile += torch.where(hit < sparse_frac, vals, torch.zeros_like(vals))
                del hit, vals
            if sigma > 0:
                tile += sigma * torch.randn(shape, generator=gen, device=dev,
                                            dtype=torch.float64)
            out[r0:r1, lo - col0:hi - col0] = tile[:, lo - blk0:hi - blk0].to(tdt)
            del tile
    return out


def gen_video_device(height=384, width=288, frames=2000, illum_rank=2, fg_size=(48, 32),
                     n_objects=3, noise=1e-3, seed=0, dtype="float32", device=None):
    """Synthetic surveillance video for the background-subtraction shape
    (BASELINE config C3), built in HBM.

    X has one column per frame (pixels in row-major order, height*width rows).
    Its parts:
      * background: a static image times 1 + a slow illumination drift of
        rank `illum_rank`; L_ref has rank 1 + illum_rank;
      * foreground: `n_objects` rectangles of `fg_size` moving at constant
        velocity (bouncing off the frame edges), with intensities that differ
        from the background — the sparse S_ref;
      * Gaussian noise of standard deviation `noise`.

    Returns (X, L_ref, fg_mask) as CUDA tensors (m x frames, fp32 / bool).
    The reference has no video generator; this one follows the paper's
    escalator / hall experiments in structure, not in pixels."""
    import torch

    dev = device or torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if dtype == "float32" else torch.float64
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    h, w, T = int(height), int(width), int(frames)
    yy = torch.linspace(0, 1, h, device=dev, dtype=torch.float64)[:, None]
    xx = torch.linspace(0, 1, w, device=dev, dtype=torch.float64)[None, :]
    # smooth static scene: a few random low-frequency waves
    bg = torch.zeros((h, w), device=dev, dtype=torch.float64)
    for _ in range(6):
        a, fy, fx, ph = torch.rand(4, generator=g, device=dev, dtype=torch.float64)
        bg += (0.2 + 0.3 * a) * torch.cos(2 * math.pi * (1 + 3 * fy) * yy +
                                          2 * math.pi * (1 + 3 * fx) * xx + 6.28 * ph)
    bg = 0.5 + 0.25 * bg / bg.abs().max()
    # illumination: spatial gain maps times slow temporal profiles
    t = torch.linspace(0, 1, T, device=dev, dtype=torch.float64)
    spatial = [bg.reshape(-1)]
    temporal = [torch.ones(T, device=dev, dtype=torch.float64)]
    for r in range(int(illum_rank)):
        gy, gx = torch.rand(2, generator=g, device=dev, dtype=torch.float64)
        spatial.append((0.1 * torch.cos(math.pi * (r + 1) * (gy * yy + gx * xx))).reshape(-1))
        temporal.append(torch.sin(2 * math.pi * (r + 1) * t + float(gy) * 3.0))
    A = torch.stack(spatial, 1)  # m x (1 + illum_rank)
    B = torch.stack(temporal, 1)  # T x (1 + illum_rank)
    L = A @ B.T
    X = L.clone()
    fg = torch.zeros((h, w, T), device=dev, dtype=torch.bool)
    Xv = X.view(h, w, T)
    oh, ow = fg_size
    iy = torch.arange(h, device=dev)[:, None, None]
    ix = torch.arange(w, device=dev)[None, :, None]
    frame = torch.arange(T, device=dev, dtype=torch.float64)
    for _ in range(int(n_objects)):
        p0y, p0x, vy, vx, val = torch.rand(5, generator=g, device=dev, dtype=torch.float64)
        ys = p0y * (h - oh) + (vy - 0.5) * 4.0 * frame
        xs = p0x * (w - ow) + (vx - 0.5) * 4.0 * frame
        # bounce: reflect the trajectory into [0, h - oh] x [0, w - ow]
        ys = (h - oh) - ((ys % (2 * (h - oh))) - (h - oh)).abs()
        xs = (w - ow) - ((xs % (2 * (w - ow))) - (w - ow)).abs()
        y0, x0 = ys.long()[None, None, :], xs.long()[None, None, :]
        box = (iy >= y0) & (iy < y0 + oh) & (ix >= x0) & (ix < x0 + ow)
        Xv.masked_fill_(box, 0.15 + 0.7 * float(val))  # later objects occlude earlier ones
        fg |= box
        del box
    if noise > 0:
        X += noise * torch.randn(X.shape, generator=g, device=dev, dtype=torch.float64)
    return X.to(tdt), L.to(tdt), fg.reshape(h * w, T)
