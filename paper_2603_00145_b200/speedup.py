"""Block-partitioned vs all-primitive rendering throughput -- the reference's
``bench_speedup`` (/root/reference/pkg/src/mgauss/cli.py:258-299), the kernel
micro-benchmark SURVEY §8(b) lists among the hot path's callers and the
reference's acceptance criterion 7 (tests/test_acceptance.py:327-337: 216k
primitives, 1M points, G = 70, r = 5, speedup >= 5).

Same inputs, same RNG stream and the same result dict; both renders run on
the device (``render_points`` through the cell-partitioned pair kernels,
``render_points_dense`` through the all-pairs kernel).  Timings are wall
clock around the host-level calls (numpy in, numpy out), as the reference
times its own, after the same 128-point warm-up.
"""

from __future__ import annotations

import time

import numpy as np


def bench_speedup(num_primitives=216000, num_points=1_000_000, grid_resolution=70, radius=5, dense_sample=10000,
                  seed=0, exact_dense=False):
    import torch

    from .core import uniform_lattice_field
    from .render import render_points, render_points_dense
    from .spatial import build

    rng = np.random.default_rng(seed)
    side = int(round(num_primitives ** (1.0 / 3.0)))
    field = uniform_lattice_field(side)
    field.positions[:] = rng.uniform(-0.98, 0.98, size=field.positions.shape)
    field.intensity_logits[:] = rng.normal(0.0, 1.0, field.count)
    field.log_scales[:] = np.log(1.0 / grid_resolution)
    grid = build(field, grid_resolution, block_radius=radius)
    points = rng.uniform(-1.0, 1.0, size=(num_points, 3))

    render_points(field, grid, None, points[:128], radius=radius)  # warm both paths before timing
    render_points_dense(field, points[:128])
    torch.cuda.synchronize()

    t0 = time.perf_counter()
    block = render_points(field, grid, None, points, radius=radius)
    torch.cuda.synchronize()
    block_time = time.perf_counter() - t0

    n_dense = num_points if exact_dense else min(dense_sample, num_points)
    t0 = time.perf_counter()
    dense = render_points_dense(field, points[:n_dense])
    torch.cuda.synchronize()
    dense_time = (time.perf_counter() - t0) * (num_points / n_dense)

    return {
        "num_primitives": field.count,
        "num_points": num_points,
        "grid_resolution": grid_resolution,
        "block_radius": radius,
        "block_seconds": block_time,
        "dense_seconds_total": dense_time,
        "dense_points_timed": n_dense,
        "speedup": dense_time / block_time,
        # not in the reference's dict: the two renders of the timed dense sample, for parity checks
        "block_intensities_sample": block.intensities[:n_dense],
        "dense_intensities_sample": dense,
        "candidate_pairs": int(np.asarray(block.contributor_counts, dtype=np.int64).sum()),
    }
