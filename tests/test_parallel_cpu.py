"""Multi-process (gloo, world_size 2, CPU) checks of the data-parallel
decomposition used by the trainer: per-rank partial accumulators over a
sharded batch, one flat all-reduce(sum), equal the full-batch totals.  The
per-rank partials come from the CPU oracle (the GPU kernels compute the same
sums on device)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2603_00145_b200.parallel import FlatAllReduce, shard_range

        z = load_golden("render_lattice12")
        g, r = int(z["g"]), int(z["r"])
        _, _, _, prec6, alpha = O.activated_parameters(z["quaternions"], z["log_scales"], z["logits"])
        cs, ci = O.build(z["positions"], g)
        rot = O.quat_to_rotation(z["t_quats"])
        lo, hi = shard_range(len(z["coords"]), rank, world)
        d_mu, d_ab, d_al, d_pts = O.block_backward(z["coords"][lo:hi], z["sids"][lo:hi], rot, z["t_trans"],
                                                   z["positions"], prec6, alpha, cs, ci, g, r, z["upstream"][lo:hi])
        # per-slice transform accumulators (sum h, sum h (x) c) for this shard
        k = len(z["t_quats"])
        acc12 = np.zeros((k, 12))
        for s in range(k):
            m = z["sids"][lo:hi] == s
            h, c = d_pts[m], z["coords"][lo:hi][m]
            acc12[s, :3] = h.sum(0)
            acc12[s, 3:] = (h[:, :, None] * c[:, None, :]).sum(0).ravel()
        loss = np.array([float(np.sum(z["upstream"][lo:hi] ** 2))])
        bufs = [torch.from_numpy(a.copy()) for a in (d_mu, d_ab, d_al, acc12, loss)]
        FlatAllReduce(bufs)()
        if rank == 0:
            out_q.put([b.numpy() for b in bufs])
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_sharded_backward_allreduce_equals_full_batch():
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=90)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    z = load_golden("render_lattice12")
    g, r = int(z["g"]), int(z["r"])
    _, _, _, prec6, alpha = O.activated_parameters(z["quaternions"], z["log_scales"], z["logits"])
    cs, ci = O.build(z["positions"], g)
    rot = O.quat_to_rotation(z["t_quats"])
    d_mu, d_ab, d_al, d_pts = O.block_backward(z["coords"], z["sids"], rot, z["t_trans"], z["positions"], prec6,
                                               alpha, cs, ci, g, r, z["upstream"])
    np.testing.assert_allclose(got[0], d_mu, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got[1], d_ab, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got[2], d_al, rtol=1e-12, atol=1e-15)
    # the reduced transform accumulators reproduce the reference transform gradients
    k = len(z["t_quats"])
    qt = O.normalize_quat(z["t_quats"])
    g_r = got[3][:, 3:].reshape(k, 3, 3)
    d_q = O.project_through_normalization(O.rotation_quat_grad(g_r, qt), z["t_quats"])
    np.testing.assert_allclose(d_q, z["d_transform"][:, :4], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got[3][:, :3], z["d_transform"][:, 4:], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got[4][0], float(np.sum(z["upstream"] ** 2)), rtol=1e-12)


def test_shard_and_slab_ranges_cover_exactly_once():
    from paper_2603_00145_b200.parallel import shard_range, slab_ranges

    for n in (0, 1, 7, 512, 65536 + 25600):
        for world in (1, 2, 3, 4, 8):
            seen = np.zeros(n, int)
            for rank in range(world):
                lo, hi = shard_range(n, rank, world)
                seen[lo:hi] += 1
            assert np.all(seen == 1)
    assert slab_ranges(512, 8)[0] == (0, 64) and slab_ranges(512, 8)[-1] == (448, 512)
