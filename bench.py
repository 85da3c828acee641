"""Benchmark: Gaussian-sample (candidate-pair) evaluations per second, forward +
backward, of the M-Gaussian training hot path on B200.

Headline workload (BASELINE.json configs[3], "C4", the configuration the
metric's 1/2/4/8-GPU figure is quoted on): 256^3 phantom at 1 mm, three
orthogonal stacks of 4 mm slices (3 x 64 x 256^2 = 12,582,912 samples), 5-tap
slab PSF, the reference's 3-level progressive schedule 0:50 -> 1000:75 ->
2000:100 over the default 4,000 iterations (train.py:56,372-381; 1M Gaussians
at the last level), a step = 65,536 batch points + one 256x256 SSIM slice.
One step = Gaussian binning + activation, point transform/PSF/binning,
forward, smooth-L1 + SSIM gradients, Gaussian-major backward, transform
gradients, fused chain-rule + aniso + Adam -- the whole device step.

The full schedule is trained (4,000 steps, ~15 s).  `value` times K steps
with inputs resident in HBM, split across the three levels in proportion to
their iteration counts (K/4, K/4, K/2: the schedule-weighted mean), each the
last steps of its level (>= W warm-up steps of that level before it).  `e2e`
is every other step of the same run through the public API
(Trainer.step_pipelined: host RNG batch -> pinned H2D -> graph replay -> loss
D2H), milestone upsampling and graph re-capture included.  Synthetic data
(paper_2603_00145_b200.synth).  C2 is reported as a secondary line.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C4|C2|C1|C3]

N > 1: one rank per GPU (re-launched under torch.distributed.run when not
already), weak scaling by default (every rank its own 65,536-point batch and
SSIM slice; NCCL all-reduce of the flat gradient buffers inside the step's
CUDA graph); --shard strong splits the reference batch instead.  Prints ONE
JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gaussian-sample evals/sec fwd+bwd"
UNIT = "pairs/s"
FLOP_FWD, FLOP_BWD = 20, 56  # algorithmic FP32 FLOP per candidate pair
SCHEDULES = {  # name -> (resolution schedule, total iterations)
    "C1": (((0, 22),), None),
    "C2": (((0, 46),), None),
    "C3": (((0, 80),), None),
    "C4": (((0, 50), (1000, 75), (2000, 100)), 4000),  # train.py:56 default length
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--shard", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="C4: W warm-up steps per level instead of the full 4,000-step schedule")
    ap.add_argument("--cpu-sample-points", type=int, default=65536)
    ap.add_argument("--no-inference", action="store_true")
    ap.add_argument("--no-recon", action="store_true", help="skip the desk64 reconstruction-to-PSNR run")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C2 line")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N-rank path with all ranks on GPU 0 (control-flow check; eager steps)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the NCCL data-parallel path even at world size 1 (exercises the N>1 code path)")
    return ap.parse_args()


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(args):
    """`bench.py --gpus N` outside torchrun: re-exec as N ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every 2 ms (nvidia-smi -lms 100 as a fallback)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_evt = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop_evt.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, int(getr(h))))
            except Exception:
                break
            self.stop_evt.wait(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nvml is not None:
            self.stop_evt.set()
            self.t.join(timeout=2)
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            sm = [float(r[0]) for r in self.rows]
            reasons = sorted({n for r in self.rows for n, b in self.BITS.items() if r[2] & b})
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.rows[0][1]), "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml, 2 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi, 100 ms"}


def peak_fp32(sm_count, mhz):
    return 2.0 * 128 * sm_count * mhz * 1e6  # FFMA = 2 FLOP, 128 FP32 lanes per SM


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}




def workload_name(name, data, cfg, psf, hw):
    from paper_2603_00145_b200.synth import CONFIGS

    dims, sp, inpl, thick, lattice, use_nrf, batch = CONFIGS[name]
    n_sl = data.num_slices
    sched = cfg.resolution_schedule
    if len(sched) > 1:
        lat = (f"progressive schedule {' -> '.join(f'{i}:{r}' for i, r in sched)} over {cfg.total_iters} iterations "
               f"(N = {', '.join(f'{r ** 3:,}' for _, r in sched)} Gaussians)")
    else:
        lat = f"N={lattice ** 3:,} Gaussians (R=G={lattice})"
    return (f"{name}: {dims}^3 @{sp}mm phantom, 3 stacks x {n_sl // 3} slices of {dims}^2 at {thick}mm, "
            f"{psf.ntaps}-tap slab PSF, {lat}, r={cfg.block_radius}"
            f"{', NRF active' if use_nrf else ''}, step = {batch:,} batch + {hw[0] * hw[1]:,} SSIM-slice points")


def make_workload(cfg_name, rank=0, final_only=False):
    """(data, cloud, slice grids, PSF, TrainConfig); final_only: a single
    level at the schedule's final resolution (tools, kernel studies)."""
    from paper_2603_00145_b200.render import SlicePSF
    from paper_2603_00145_b200.synth import CONFIGS, make_config
    from paper_2603_00145_b200.train import TrainConfig

    data = make_config(cfg_name, seed=7)
    _, _, _, _, lattice, use_nrf, batch = CONFIGS[cfg_name]
    sched, total = SCHEDULES.get(cfg_name, (((0, lattice),), None))
    if final_only:
        sched, total = ((0, sched[-1][1]),), None
    grids = []
    for k in range(data.num_slices):
        c, t = data.slice_grid(k)
        grids.append(type("SG", (), {"coords": c, "target": t, "slice_id": k})())
    psf = SlicePSF(data.psf_offsets, data.psf_weights, data.through_dirs)
    # NRF configs (C3) measure the refinement phase: the residual field is active from the first step
    cfg = TrainConfig(resolution_schedule=sched, use_nrf=use_nrf, nrf_activation_iter=0, use_ssim=True,
                      batch_points=batch, seed=7, total_iters=total or 10 ** 9)
    cloud = type("Cloud", (), {"coords": data.coords, "intensities": data.intensities,
                               "slice_ids": data.slice_ids})()
    return data, cloud, grids, psf, cfg


def split_steps(k, sched, total):
    """K timed steps over the levels in proportion to their iteration counts."""
    if len(sched) == 1:
        return [k]
    its = [b - a for (a, _), (b, _) in zip(sched, list(sched[1:]) + [(total, None)])]
    raw = [k * i / sum(its) for i in its]
    ks = [max(1, int(round(x))) for x in raw]
    while sum(ks) > k and max(ks) > 1:
        ks[int(np.argmax(ks))] -= 1
    while sum(ks) < k:
        ks[int(np.argmax(np.array(raw) - np.array(ks)))] += 1
    return ks


def _allsum(x, dist_on, op="sum"):
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    if dist_on:
        import torch.distributed as tdist

        tdist.all_reduce(t, op=tdist.ReduceOp.MAX if op == "max" else tdist.ReduceOp.SUM)
    return float(t.item())


def timed_window(tr, k, dist_on):
    """k steps with their indices pre-drawn from the trainer's RNG stream and
    resident on the device; CUDA events on the launching stream, barrier +
    synchronize on both sides.  -> (ms, pairs, h2d bytes per step)."""
    import torch

    steps = [tr.draw_step() for _ in range(k)]
    plan = steps[0][1]
    dev = [torch.from_numpy(a).cuda() for a, _ in steps]
    B = tr._buffers(plan)
    torch.cuda.synchronize()
    p0 = int(B.pairs.item())
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for (_, pl), ix in zip(steps, dev):
        tr.load_indices(ix, pl)
        tr.run_device_step(pl)
        tr.iteration += 1
    e1.record()
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    return e0.elapsed_time(e1), int(B.pairs.item()) - p0, int(dev[0].numel() * 8), plan


def pipelined_segment(tr, n):
    """n steps through the public API (host RNG batch, pinned H2D, graph
    replay, loss D2H every step), wall-clocked.  -> (seconds, pairs)."""
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bufs = []
    for _ in range(n):
        tr.step_pipelined()
        if not bufs or bufs[-1] is not tr._bufs:
            bufs.append(tr._bufs)
    tr.flush()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return dt, bufs


def kernel_times(tr, n=3):
    """Average device time of the forward and backward pair kernels and the
    fused update, via CUDA events on the launching (current) stream, over n
    eager steps of the trainer's current level."""
    import torch

    from paper_2603_00145_b200 import _native as N

    L = N.lib()
    fwd, bwd, upd, pairs, launches = [], [], [], [], []
    orig = L.mg_forward, L.mg_backward, L.mg_gauss_update_inv, L.mg_gauss_update

    class Timed:
        def __init__(self, fn, sink):
            self.fn, self.sink = fn, sink

        def __call__(self, *a):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = self.fn(*a)
            e1.record()
            self.sink.append((e0, e1))
            return rc

    try:
        L.mg_forward, L.mg_backward = Timed(orig[0], fwd), Timed(orig[1], bwd)
        L.mg_gauss_update_inv, L.mg_gauss_update = Timed(orig[2], upd), Timed(orig[3], upd)
        for _ in range(n):
            all_idx, plan = tr.draw_step()
            B = tr.load_indices(torch.from_numpy(all_idx).cuda(), plan)
            c0 = L.mg_launch_count()
            tr._body(B, plan)
            launches.append(L.mg_launch_count() - c0)
            torch.cuda.synchronize()
            pairs.append(int(B.cnt.sum().item()))
    finally:
        L.mg_forward, L.mg_backward, L.mg_gauss_update_inv, L.mg_gauss_update = orig
    torch.cuda.synchronize()
    return {"forward_ms": float(np.mean([a.elapsed_time(b) for a, b in fwd])),
            "backward_ms": float(np.mean([a.elapsed_time(b) for a, b in bwd])),
            "update_ms": float(np.mean([a.elapsed_time(b) for a, b in upd])),
            "pairs_per_launch": float(np.mean(pairs)), "launches_per_step": int(max(launches))}


def parity_check(tr, data, psf, npts=4096, seed=11):
    """Parity of the benchmarked kernels on the benchmarked (trained) field:
    render_points + render_backward (float32 device path, PSF) on npts batch
    points of the current level against the CPU oracle (oracle.psf_render /
    psf_backward, float64) -- SURVEY §8(c) tolerances."""
    from oracle import oracle as O
    from paper_2603_00145_b200.render import render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    f = tr.field.to_host()
    ts = tr.transforms_host()
    g, r = tr.field.resolution, tr.config.block_radius
    rng = np.random.default_rng(seed)
    idx = rng.choice(data.coords.shape[0], npts, replace=False)
    coords, sids = data.coords[idx], data.slice_ids[idx]
    up = rng.normal(size=npts) * 1e-3

    class Bt:
        pass

    bt = Bt()
    bt.coords, bt.slice_ids = coords, sids
    grid = build(f, g, r)
    out = render_points(f, grid, ts, bt, slice_psf=psf)
    gr = render_backward(f, grid, ts, bt, up, slice_psf=psf)
    thr = min(16, os.cpu_count() or 1)
    inten, cnt = O.psf_render(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, sids,
                              ts.quats, ts.translations, psf.offsets, psf.weights, psf.through_dirs, thr)
    og = O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, sids, ts.quats,
                        ts.translations, psf.offsets, psf.weights, psf.through_dirs, up, thr)
    rel = np.abs(out.intensities - inten) / np.maximum(np.abs(inten), 1e-30)
    grads = {}
    ok = bool(np.array_equal(out.contributor_counts, cnt)) and bool(np.all(rel <= 1e-4))
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params"):
        a, w = getattr(gr, name), getattr(og, name)
        tol = 1e-4 * np.abs(w) + 1e-6 * np.abs(w).max()
        worst = float(np.max(np.abs(a - w) / np.maximum(tol, 1e-300)))
        grads[name] = worst
        ok = ok and worst <= 1.0
    return {"ok": ok, "points": npts, "taps": psf.ntaps, "pairs": int(cnt.sum()),
            "counts_bit_exact": bool(np.array_equal(out.contributor_counts, cnt)),
            "max_rel_intensity": float(rel.max()), "grad_err_over_tol": grads,
            "field": f"trained level-{g} field at iteration {tr.iteration}",
            "tolerance": "counts exact; I rel 1e-4; grads |d| <= 1e-4|ref| + 1e-6 max|ref| (SURVEY §8(c))"}


def cpu_pairs_baseline(tr, data, psf, sample_points, threads):
    """Reference CPU arm on the same field: the oracle's C restatement of
    _kernels.block_forward + block_backward (the reference's numba kernels,
    render.py:161-187,276-317 with `prepared`), all host threads, on
    `sample_points` batch points x PSF taps of the benchmarked level.  The
    O(N) activation/binning (prepared) is outside the timed region, as is
    the reference's O(N) numpy epilogue: this is the reference's pair
    throughput, an upper bound on its whole-step pairs/s."""
    from oracle import oracle as O

    f = tr.field.to_host()
    ts = tr.transforms_host()
    g, r = tr.field.resolution, tr.config.block_radius
    return _cpu_pairs(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, ts, data, psf,
                      sample_points, threads, np.random.default_rng(3), O)


def _cpu_pairs(pos, quat, ls, lg, g, r, ts, data, psf, npts, threads, rng, O):
    _, _, _, prec6, alpha = O.activated_parameters(quat, ls, lg)
    cs, ci = O.build(pos, g)
    rot = O.quat_to_rotation(ts.quats)
    idx = rng.choice(data.coords.shape[0], npts, replace=False)
    coords, sids = data.coords[idx], data.slice_ids[idx]
    dirs = np.asarray(psf.through_dirs).reshape(-1, 3)
    shift = dirs[np.clip(sids, 0, None)] * (sids >= 0)[:, None]
    pts = np.ascontiguousarray(np.concatenate([coords + o * shift for o in psf.offsets]))
    ps = np.concatenate([sids] * psf.ntaps)
    up = np.concatenate([w * rng.normal(size=npts) * 1e-3 for w in psf.weights])
    t0 = time.perf_counter()
    _, cnt, _ = O.block_forward(pts, ps, rot, ts.translations, pos, prec6, alpha, cs, ci, g, r, threads)
    O.block_backward(pts, ps, rot, ts.translations, pos, prec6, alpha, cs, ci, g, r, up, threads)
    dt = time.perf_counter() - t0
    pairs = int(cnt.sum())
    return pairs / dt, pairs, dt


def run_ours(args):
    import torch

    rank, world, local = dist_info()
    if args.backend == "gloo":  # control-flow check of the N-rank path on a one-GPU box (ranks share GPU 0)
        local = 0
    torch.cuda.set_device(local)
    group = None
    dist_on = world > 1 or args.force_dist
    if dist_on:
        import torch.distributed as tdist

        if not tdist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            if args.backend == "gloo":
                tdist.init_process_group("gloo", rank=rank, world_size=world)
            else:
                tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        group = tdist.group.WORLD
    from paper_2603_00145_b200 import _native as N
    from paper_2603_00145_b200.train import Trainer, freeze_gc

    freeze_gc()
    data, cloud, grids, psf, cfg = make_workload(args.config, rank)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=not args.no_graph,
                 dist=group, shard=args.shard)
    sched = cfg.resolution_schedule
    total = SCHEDULES.get(args.config, (None, None))[1]
    multilevel = total is not None
    ks = split_steps(args.steps, sched, total) if multilevel else [args.steps]
    W = max(args.warmup, 3)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    levels = []
    e2e_t, e2e_pairs, e2e_steps = 0.0, 0.0, 0
    h2d = 0
    for li, (it0, res) in enumerate(sched):
        it_end = sched[li + 1][0] if li + 1 < len(sched) else (total if multilevel else it0 + W + ks[li])
        k = ks[li]
        n_seg = (it_end - k) - it0 if (multilevel and not args.quick) else W
        if multilevel and args.quick:
            tr.iteration = it0
        if not multilevel:
            # single-level configs: W warm-up steps (first-touch, graph capture) are not part of the e2e
            # number; the e2e segment is then a steady-state run of its own
            pipelined_segment(tr, W)
            n_seg = max(50, k)
        dt, bufs = pipelined_segment(tr, n_seg)
        seg_pairs = sum(int(b.pairs.item()) for b in bufs)
        e2e_t += _allsum(dt, dist_on, "max")
        e2e_pairs += _allsum(seg_pairs, dist_on)
        e2e_steps += n_seg
        ms, pairs, h2d, plan = timed_window(tr, k, dist_on)
        ms_max = _allsum(ms, dist_on, "max")
        pairs_all = _allsum(pairs, dist_on)
        kt = kernel_times(tr)  # every rank: the eager steps carry the step's collectives
        levels.append({"level": li, "resolution": res, "gaussians": res ** 3, "iterations": [it0, it_end],
                       "timed_steps": k, "ms": ms_max, "ms_per_step": ms_max / k, "pairs_per_step": pairs_all / k,
                       "value": pairs_all / (ms_max / 1e3), "kernels": kt,
                       "e2e_segment": {"steps": n_seg, "seconds": dt, "pairs": seg_pairs}})
    clocks = sampler.stop()
    ms_tot = sum(lv["ms"] for lv in levels)
    pairs_tot = sum(lv["pairs_per_step"] * lv["timed_steps"] for lv in levels)
    value = pairs_tot / (ms_tot / 1e3)
    e2e_val = e2e_pairs / e2e_t if e2e_t > 0 else None
    hw = plan.hw
    wl = workload_name(args.config, data, cfg, psf, hw)
    graph_used = tr._graph is not None
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = parity_check(tr, data, psf)
        except Exception as exc:
            parity = {"ok": False, "error": repr(exc)[:300]}
    cpu = None
    if world == 1:  # the CPU baseline is an N = 1 figure
        threads = os.cpu_count() or 1
        v, p, dt = cpu_pairs_baseline(tr, data, psf, args.cpu_sample_points, threads)
        v1, p1, dt1 = cpu_pairs_baseline(tr, data, psf, max(1024, args.cpu_sample_points // 16), 1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{args.cpu_sample_points} batch points x {psf.ntaps} PSF taps on the final "
                         f"{tr.field.resolution}^3 level's trained field ({p} pairs, {dt:.1f} s): "
                         f"oracle C block_forward + block_backward (the reference's kernels, prepared inputs)",
               "value_1thread": v1, "sample_1thread": f"{max(1024, args.cpu_sample_points // 16)} points "
                                                      f"({p1} pairs, {dt1:.1f} s)"}
    tr.close()
    del tr
    torch.cuda.empty_cache()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    peaks = load_peaks()
    sms = N.lib().mg_device_sm_count()
    mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak = peak_fp32(sms, mhz)
    # schedule-weighted kernel roofline: sum_l w_l pairs_l (20 + 56) / sum_l w_l (t_fwd + t_bwd)
    wts = [lv["timed_steps"] for lv in levels]
    kp = sum(w * lv["kernels"]["pairs_per_launch"] for w, lv in zip(wts, levels))
    kf = sum(w * lv["kernels"]["forward_ms"] for w, lv in zip(wts, levels))
    kb = sum(w * lv["kernels"]["backward_ms"] for w, lv in zip(wts, levels))
    achieved = kp * (FLOP_FWD + FLOP_BWD) / ((kf + kb) / 1e3)
    last = levels[-1]["kernels"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"r02_traffic_{args.config}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp))
        except Exception:
            traffic = None
    nlaunch = max(lv["kernels"]["launches_per_step"] for lv in levels)
    secondary = None
    if not args.no_secondary and args.config != "C2" and world == 1:
        try:
            secondary = secondary_line("C2", args)
        except Exception as exc:
            secondary = {"error": repr(exc)[:200]}
        torch.cuda.empty_cache()
    infer = None
    if not args.no_inference:
        try:
            infer = inference_c5()
        except Exception as exc:  # report, never fail the training bench
            infer = {"error": repr(exc)[:200]}
        torch.cuda.empty_cache()
    recon = None
    if not args.no_recon:
        try:
            recon = recon_desk64()
        except Exception as exc:
            recon = {"error": repr(exc)[:200]}
    speed = None
    if not args.no_recon and world == 1:
        try:
            speed = speedup_c7()
        except Exception as exc:
            speed = {"error": repr(exc)[:200]}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_tot / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.shard == "weak" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl, "global_batch": cfg.batch_points * (world if args.shard == "weak" else 1),
                   "pairs_per_step": pairs_tot / args.steps, "parallelism": f"dp{world}",
                   "timed_steps_per_level": ks, "full_schedule_trained": multilevel and not args.quick,
                   "l2": "inputs larger than L2: every step gathers its batch at fresh random indices from the "
                         "device sample pool (12.6M samples, 600+ MiB for C4; L2 126 MB); the model state stays "
                         "L2-resident across steps as in training",
                   "cuda_graph": graph_used, "shard": args.shard},
        "levels": levels,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 32 + 4,
                "steps": e2e_steps,
                "path": ("Trainer.step_pipelined() over every untimed step of the schedule run: host RNG batch -> "
                         "pinned H2D -> graph replay -> async loss D2H; milestone upsampling and graph "
                         "re-capture included") if multilevel else
                        ("Trainer.step_pipelined(), steady state after the warm-up steps: host RNG batch -> pinned "
                         "H2D -> graph replay -> async loss D2H")},
        "roofline": {"bound": "fp32", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"nominal 256 FLOP/clk/SM x {sms} SMs x {mhz:.0f} MHz (measured SM clock); "
                                    "MEASURED_PEAKS.json has no FP32 figure",
                     "accounting": f"pair kernels forward ({FLOP_FWD} FLOP/pair) + backward ({FLOP_BWD} FLOP/pair), "
                                   "schedule-weighted over the levels, CUDA-event kernel times",
                     "kernels_last_level": {
                         "forward": {"ms": last["forward_ms"],
                                     "frac": last["pairs_per_launch"] * FLOP_FWD / (last["forward_ms"] / 1e3) / peak},
                         "backward": {"ms": last["backward_ms"],
                                      "frac": last["pairs_per_launch"] * FLOP_BWD / (last["backward_ms"] / 1e3) / peak},
                         "update_ms": last["update_ms"], "pairs_per_launch": last["pairs_per_launch"]}},
        "parity": parity,
        "cpu_baseline": cpu,
        "secondary": secondary,
        "inference": infer,
        "recon": recon,
        "block_speedup": speed,
        "clocks": clocks,
        "gpu_launches": nlaunch * args.steps,
        "gpu_launches_note": "library kernels per step (mg_launch_count over one eager step) x timed steps; "
                             "torch fill/copy plumbing kernels not counted",
    }
    print(json.dumps(out))
    if dist_on:
        torch.distributed.destroy_process_group()


def secondary_line(name, args, steps=20):
    """One-level config (C2) at N = 1: the round-1 headline, kept for continuity."""
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = make_workload(name, 0)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    try:
        dt, bufs = pipelined_segment(tr, max(args.warmup, 3) + 30)
        e2e_pairs = int(tr._bufs.pairs.item())
        ms, pairs, _, plan = timed_window(tr, steps, False)
        kt = kernel_times(tr)
        e2e_steps = max(args.warmup, 3) + 30
    finally:
        tr.close()
    peak = peak_fp32(148, 1965.0)
    return {"workload": workload_name(name, data, cfg, psf, plan.hw), "value": pairs / (ms / 1e3),
            "ms_per_step": ms / steps, "pairs_per_step": pairs / steps,
            "e2e_incl_capture": {"value": e2e_pairs / dt, "steps": e2e_steps},
            "kernels": kt, "frac_pair_kernels": kt["pairs_per_launch"] * (FLOP_FWD + FLOP_BWD) /
            ((kt["forward_ms"] + kt["backward_ms"]) / 1e3) / peak}


def run_reference(args):
    """Reference arm: the reference's pair kernels (block_forward +
    block_backward, _kernels.py:24-144, as the oracle's C restatement -- the
    reference itself is Python + numba and cannot travel to the GPU box) on
    the host cores, same config and metric, each step a bounded sample of the
    workload: per level of the schedule, the level's initial lattice field
    and the same split of K steps across the levels as our arm."""
    rank, world, _ = dist_info()
    if rank != 0:
        return
    import torch  # noqa: F401  (workload generator imports it)

    from oracle import oracle as O
    from paper_2603_00145_b200.core import uniform_lattice_field

    threads = os.cpu_count() or 1
    data, cloud, grids, psf, cfg = make_workload(args.config, 0)
    sched = cfg.resolution_schedule
    total = SCHEDULES.get(args.config, (None, None))[1]
    ks = split_steps(args.steps, sched, total) if total else [args.steps]
    per_step = max(1024, min(args.cpu_sample_points, 16384))
    rng = np.random.default_rng(7)
    total_pairs, total_t = 0, 0.0
    for (it0, res), k in zip(sched, ks):
        f = uniform_lattice_field(res)
        f.intensity_logits[:] = O.init_logits(data.coords, data.intensities, res)
        for s in range(max(1, args.warmup // len(sched)) + k):
            v, p, dt = _cpu_pairs(f.positions, f.quaternions, f.log_scales, f.intensity_logits, res, 5,
                                  data.transforms, data, psf, per_step, threads, rng, O)
            if s >= max(1, args.warmup // len(sched)):
                total_pairs += p
                total_t += dt
    v = total_pairs / total_t
    hw = grids[0].target.shape
    sample = (f"{per_step} batch points x {psf.ntaps} PSF taps per step on each level's lattice field "
              f"(K split across levels {ks}); block_forward + block_backward with prepared inputs")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, data, cfg, psf, np.asarray(hw)), "cpu_threads": threads},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def speedup_c7():
    """The reference's bench_speedup at its acceptance-criterion-7 inputs (cli.py:258-299,
    tests/test_acceptance.py:327-337): 216k primitives, 1M points, G = 70, r = 5, seed 7, wall clock around the
    host-level render_points / render_points_dense calls (numpy in and out), as the reference times them."""
    from paper_2603_00145_b200.speedup import bench_speedup

    row = bench_speedup(num_primitives=216000, num_points=1_000_000, grid_resolution=70, radius=5,
                        dense_sample=10000, seed=7)
    b, d = row.pop("block_intensities_sample"), row.pop("dense_intensities_sample")
    row["block_vs_dense_max_rel"] = float(np.abs(b - d).max() / max(np.abs(d).max(), 1e-30))
    row["block_pairs_per_s"] = row["candidate_pairs"] / row["block_seconds"]
    row["reference"] = {"block_seconds": 64.3, "dense_seconds_total": 1007.0, "threads": 1,
                        "source": "BASELINE.md section 2 (survey measurement of the reference, not published)"}
    row["vs_reference_block"] = 64.3 / row["block_seconds"]
    return row


def recon_desk64():
    """BASELINE "recon s to PSNR": the reference's desk-scale reconstruction
    (configs/desk64.cfg: 64^3 phantom, 1500 iterations, lattice 16^3 -> 48^3,
    NRF from 600, SSIM) on the cloud the reference devoxelised, recorded with
    the reference's own PSNR and wall time by tests/golden/make_recon.py."""
    import torch

    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.train import Trainer

    path = os.path.join(ROOT, "tests", "golden", "recon_desk64.npz")
    if not os.path.exists(path):
        return None
    cloud, ts, grids, cfg, tgt = load_recon_fixture(path)
    runs = []
    for _ in range(2):  # cold (first in the process: lazy kernel loading), then warm
        tr = Trainer(cloud, ts, cfg, slice_grids=grids, graph=True)
        try:
            runs.append(reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale))
        finally:
            tr.close()
        del tr
        torch.cuda.empty_cache()
    (vol, t_train, t_total), cold = runs[1], runs[0]
    db = psnr(vol.astype(np.float64), tgt.gt.astype(np.float64))
    assert np.array_equal(vol, cold[0]), "reconstruction is not deterministic"
    return {"workload": f"desk64: 64^3 nested-ellipsoids, 3 stacks x 16 slices at 4 mm, {cfg.total_iters} iters, "
                        f"lattice {cfg.resolution_schedule[0][1]}^3 -> {cfg.final_resolution}^3, NRF@"
                        f"{cfg.nrf_activation_iter}, batch {cfg.batch_points} + SSIM slice",
            "train_seconds": t_train, "seconds_incl_volume": t_total, "psnr_db": db,
            "train_seconds_cold": cold[1],
            "timing": "second of two identical runs in the process (the first, cold, pays lazy CUDA module "
                      "loading and first graph captures); both give the bit-identical volume",
            "reference_psnr_db": tgt.ref_psnr_db, "reference_train_seconds": tgt.ref_seconds,
            "reference_threads": tgt.ref_threads}


def _c5_field(kind, R=126):
    """C5 fields (SURVEY §8(d) option 2, seed 7): lattice positions + N(0, 0.1/R) jitter, identity + N(0, 0.1)
    quaternions, log-scales log(1/R) + N(0, 0.1), logits N(0, 1).  'drifted' jitters by half a cell (cell
    occupancy 0..4, like a trained field); 'clustered' squeezes the field into the central eighth (~8 Gaussians
    per occupied cell: every central tile overflows the shared-memory staging -> the global-walk path)."""
    from paper_2603_00145_b200.core import lattice_node_positions

    n = R ** 3
    rng = np.random.default_rng(7)
    sig = {"lattice": 0.1, "drifted": 0.5, "clustered": 0.1}[kind]
    pos = lattice_node_positions(R) + rng.normal(0, sig / R, (n, 3))
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    q += rng.normal(0, 0.1, (n, 4))
    ls = np.log(1.0 / R) + rng.normal(0, 0.1, (n, 3))
    lg = rng.normal(0, 1, n)
    if kind == "clustered":
        pos *= 0.5
        ls += np.log(0.5)
    return pos, q, ls, lg


def _c5_time(pos, q, ls, lg, R, reps):
    import torch

    from paper_2603_00145_b200 import _native as N
    from paper_2603_00145_b200.render import sample_volume_device
    from paper_2603_00145_b200.spatial import build_device

    n = pos.shape[0]
    dev = torch.device("cuda")
    pos_d = torch.from_numpy(pos).float().to(dev)
    q_d = torch.from_numpy(q).float().to(dev)
    ls_d = torch.from_numpy(ls).float().to(dev)
    lg_d = torch.from_numpy(lg).float().to(dev)
    L = N.lib()
    d = build_device(pos_d, R)
    grec = torch.empty((n, 12), dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(L.mg_activate(N.ptr(pos_d), N.ptr(q_d), N.ptr(ls_d), N.ptr(lg_d), n, N.ptr(d["order"]), N.ptr(grec),
                          N.ptr(err), N.stream_ptr()))
    dims = (512, 512, 512)
    bounds = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    out = sample_volume_device(grec, n, d["starts"], R, 5, dims, bounds)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = sample_volume_device(grec, n, d["starts"], R, 5, dims, bounds)
    e1.record()
    torch.cuda.synchronize()
    del out
    ms = e0.elapsed_time(e1) / reps
    # exact candidate-pair count: sum over voxels of the Gaussians within Chebyshev 5 cells of the voxel's cell
    starts = d["starts"].cpu().numpy().astype(np.int64)
    cnt = np.diff(starts).reshape(R, R, R)
    ps = np.zeros((R + 1, R + 1, R + 1), np.int64)
    ps[1:, 1:, 1:] = cnt.cumsum(0).cumsum(1).cumsum(2)
    lo = np.clip(np.arange(R) - 5, 0, R)
    hi = np.clip(np.arange(R) + 6, 0, R)
    I0, J0, K0 = np.meshgrid(lo, lo, lo, indexing="ij")
    I1, J1, K1 = np.meshgrid(hi, hi, hi, indexing="ij")
    cand = (ps[I1, J1, K1] - ps[I0, J1, K1] - ps[I1, J0, K1] - ps[I1, J1, K0] + ps[I0, J0, K1] + ps[I0, J1, K0]
            + ps[I1, J0, K0] - ps[I0, J0, K0])
    ax = -1.0 + np.arange(512) * (2.0 / 511)
    vc = np.bincount(np.clip(np.floor((ax + 1.0) * (R / 2.0)).astype(np.int64), 0, R - 1), minlength=R)
    pairs = float(np.einsum("i,j,k,ijk->", vc, vc, vc, cand.astype(np.float64)))
    peak = peak_fp32(L.mg_device_sm_count(), 1965.0)
    return {"ms": ms, "voxels_per_s": 512 ** 3 / (ms / 1e3), "pairs_per_s": pairs / (ms / 1e3), "pairs": pairs,
            "roofline_frac_fp32": pairs * FLOP_FWD / (ms / 1e3) / peak,
            "max_gaussians_per_cell": int(cnt.max()), "occupied_cells": float((cnt > 0).mean())}


def inference_c5(reps=3):
    """C5 (BASELINE.json configs[4]): sample a 512^3 node-inclusive volume over
    [-1, 1]^3 from a 2,000,376-Gaussian field (R = G = 126, r = 5): the headline
    numbers on the jittered lattice, plus a drifted and a clustered field."""
    R = 126
    out = {"workload": "C5: 512^3 volume from 2,000,376 Gaussians (R=G=126, r=5), synthetic lattice field"}
    out.update(_c5_time(*_c5_field("lattice", R), R, reps))
    out["other_fields"] = {k: _c5_time(*_c5_field(k, R), R, max(1, reps - 1)) for k in ("drifted", "clustered")}
    return out


def main():
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ:
        relaunch_distributed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
