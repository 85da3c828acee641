"""Per-kernel device time of one eager C3 step (NRF active): python tools/nrf_prof.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload("C3", 0)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=False)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            tr.step()
        torch.cuda.synchronize()
    rows = []
    for e in prof.key_averages():
        if e.device_time_total > 0:
            rows.append((e.device_time_total / 3.0, e.count // 3, e.key[:90]))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"total device us/step {tot:.0f}")
    for t, c, k in rows[:30]:
        print(f"{t:9.1f} us  x{c:3d}  {k}")


if __name__ == "__main__":
    main()
