"""Wall-time profile of the desk64 reconstruction: seconds per 100-step
window (device synchronised at each window edge), to find where recon time
goes (milestones, graph captures, host stalls).

    python tools/recon_prof.py [--graph 1] [--repeat 2]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--cprofile", type=int, default=-1, help="cProfile this run index")
    ap.add_argument("--phases", type=int, default=1, help="synchronised timing of milestone phases")
    ap.add_argument("--nogc", type=int, default=0, help="disable the Python cyclic GC")
    a = ap.parse_args()
    import torch

    import gc

    if a.nogc:
        gc.disable()
    gc_log = []
    gc_t = {}

    def _gc_cb(phase, info):
        if phase == "start":
            gc_t["t"] = time.perf_counter()
        else:
            dt = time.perf_counter() - gc_t.get("t", time.perf_counter())
            if dt > 0.005:
                gc_log.append((info["generation"], round(dt, 4), info["collected"]))

    gc.callbacks.append(_gc_cb)

    from paper_2603_00145_b200.recon import load_recon_fixture
    from paper_2603_00145_b200.train import Trainer

    phase_log = []
    if a.phases:
        def timed(name, fn):
            def w(*args, **kw):
                if torch.cuda.is_current_stream_capturing():
                    return fn(*args, **kw)
                torch.cuda.synchronize()
                t = time.perf_counter()
                out = fn(*args, **kw)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                if dt > 0.005:
                    phase_log.append((name, round(dt, 4)))
                return out
            return w
        for nm in ("_apply_milestones", "_capture", "_body", "load_indices", "_buffers", "_next_batch"):
            setattr(Trainer, nm, timed(nm, getattr(Trainer, nm)))
    cloud, ts, grids, cfg, tgt = load_recon_fixture(os.path.join(ROOT, "tests", "golden", "recon_desk64.npz"))
    for rep in range(a.repeat):
        t_init = time.perf_counter()
        tr = Trainer(cloud, ts, cfg, slice_grids=grids, graph=bool(a.graph))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        print(f"run {rep}: init {t0 - t_init:.3f}s", flush=True)
        last = t0
        win = []
        prof = None
        if rep == a.cprofile:
            import cProfile
            prof = cProfile.Profile()
            prof.enable()
        while tr.iteration < cfg.total_iters:
            tr.step(sync=False)
            if tr.iteration % 100 == 0 or tr.iteration in (1, 2, 3):
                torch.cuda.synchronize()
                now = time.perf_counter()
                win.append((tr.iteration, tr.field.count, round(now - last, 4)))
                last = now
        torch.cuda.synchronize()
        if prof is not None:
            import pstats
            prof.disable()
            pstats.Stats(prof).sort_stats("cumulative").print_stats(30)
        print(f"run {rep}: train {time.perf_counter() - t0:.3f}s", win, flush=True)
        if phase_log:
            print(f"run {rep}: phases > 5 ms", phase_log, flush=True)
            phase_log.clear()
        print(f"run {rep}: gc collections > 5 ms (gen, s, collected) {gc_log}; tracked objects "
              f"{len(gc.get_objects())}, frozen {gc.get_freeze_count()}", flush=True)
        gc_log.clear()
        tr.close()
        del tr


if __name__ == "__main__":
    main()
