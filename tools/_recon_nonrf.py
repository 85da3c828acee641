import os, sys, time, dataclasses
sys.path.insert(0, "/root/repo")
import torch
from paper_2603_00145_b200.recon import load_recon_fixture
from paper_2603_00145_b200.train import Trainer
cloud, ts, grids, cfg, tgt = load_recon_fixture("/root/repo/tests/golden/recon_desk64.npz")
for nrf_at in (cfg.nrf_activation_iter, 10**9, cfg.nrf_activation_iter):
    c = dataclasses.replace(cfg, nrf_activation_iter=nrf_at)
    tr = Trainer(cloud, ts, c, slice_grids=grids, graph=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); last = t0; win = []
    while tr.iteration < c.total_iters:
        tr.step(sync=False)
        if tr.iteration % 100 == 0:
            torch.cuda.synchronize(); now = time.perf_counter(); win.append(round(1e3 * (now - last) / 100, 3)); last = now
    torch.cuda.synchronize()
    print(nrf_at, "train %.3f s" % (time.perf_counter() - t0), "ms/step per 100:", win, flush=True)
    tr.close(); del tr
