"""Benchmark: Gaussian-sample (candidate-pair) evaluations per second, forward +
backward, for one training step of the M-Gaussian hot path on B200.

Workload (BASELINE.json configs[1], "C2"): 160^3 phantom at 0.8 mm, three
orthogonal stacks of 3 mm slices (3 x 42 x 160^2 = 3,225,600 samples), 3-tap
Gaussian slice PSF, 100k Gaussians (R = G = 46 lattice, N = 97,336), a step =
65,536 batch points + one 160x160 SSIM slice, each expanded to 3 PSF taps.
One step = Gaussian binning + activation, point transform/binning, forward,
smooth-L1 + SSIM gradients, Gaussian-major backward, transform gradients,
fused chain-rule + aniso + Adam.  Synthetic data (paper_2603_00145_b200.synth).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 is launched with torch.distributed.run: one rank per GPU, weak scaling
(each rank its own 65,536-point batch), NCCL all-reduce of the per-Gaussian
gradient accumulators.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
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
CONFIG = "C2"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-sample-points", type=int, default=65536)
    ap.add_argument("--no-inference", action="store_true")
    ap.add_argument("--no-recon", action="store_true", help="skip the desk64 reconstruction-to-PSNR run")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the NCCL data-parallel path even at world size 1 (exercises the N>1 code path)")
    return ap.parse_args()


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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


def workload_name(name, data, cfg, psf, hw):
    from paper_2603_00145_b200.synth import CONFIGS

    dims, sp, inpl, thick, lattice, use_nrf, batch = CONFIGS[name]
    n_sl = data.num_slices
    return (f"{name}: {dims}^3 @{sp}mm phantom, 3 stacks x {n_sl // 3} slices of {dims}^2 at {thick}mm, "
            f"{psf.ntaps}-tap slab PSF, N={lattice ** 3:,} Gaussians (R=G={lattice}), r={cfg.block_radius}"
            f"{', NRF active' if use_nrf else ''}, step = {batch:,} batch + {hw[0] * hw[1]:,} SSIM-slice points")


def make_workload(cfg_name, rank):
    from paper_2603_00145_b200.render import SlicePSF
    from paper_2603_00145_b200.synth import CONFIGS, make_config
    from paper_2603_00145_b200.train import TrainConfig

    data = make_config(cfg_name, seed=7)
    _, _, _, _, lattice, use_nrf, batch = CONFIGS[cfg_name]
    grids = []
    for k in range(data.num_slices):
        c, t = data.slice_grid(k)
        grids.append(type("SG", (), {"coords": c, "target": t, "slice_id": k})())
    psf = SlicePSF(data.psf_offsets, data.psf_weights, data.through_dirs)
    # NRF configs (C3) measure the refinement phase: the residual field is active from the first step
    cfg = TrainConfig(resolution_schedule=((0, lattice),), use_nrf=use_nrf, nrf_activation_iter=0, use_ssim=True,
                      batch_points=batch, seed=7 + rank, total_iters=10 ** 9)
    cloud = type("Cloud", (), {"coords": data.coords, "intensities": data.intensities,
                               "slice_ids": data.slice_ids})()
    return data, cloud, grids, psf, cfg


def peak_fp32(sm_count, mhz):
    return 2.0 * 128 * sm_count * mhz * 1e6  # FFMA = 2 FLOP, 128 FP32 lanes per SM


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def count_graph_kernels(graph):
    """Kernel nodes in a captured torch CUDA graph (cudaGraphGetNodes + node types)."""
    try:
        import ctypes

        raw = graph.raw_cuda_graph()
        rt = ctypes.CDLL("libcudart.so")
    except Exception:
        try:
            import ctypes
            import glob

            import torch

            libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
            libs += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
            rt = ctypes.CDLL(libs[0])
            raw = graph.raw_cuda_graph()
        except Exception:
            return None
    n = ctypes.c_size_t(0)
    if rt.cudaGraphGetNodes(ctypes.c_void_p(raw), None, ctypes.byref(n)) != 0:
        return None
    nodes = (ctypes.c_void_p * n.value)()
    rt.cudaGraphGetNodes(ctypes.c_void_p(raw), nodes, ctypes.byref(n))
    kernels = 0
    for i in range(n.value):
        t = ctypes.c_int(0)
        rt.cudaGraphNodeGetType(ctypes.c_void_p(nodes[i]), ctypes.byref(t))
        kernels += int(t.value == 0)  # cudaGraphNodeTypeKernel
    return kernels


def cpu_baseline(trainer, data, psf, sample_points, threads):
    """Oracle (C restatement of the reference kernels + numpy host math), all host
    threads, on a bounded sample of one step: render + backward over the first
    `sample_points` batch points with the same field, transforms and PSF."""
    from oracle import oracle as O

    f = trainer.field.to_host()
    ts = trainer.transforms_host()
    g = trainer.field.resolution
    idx = trainer._next_batch()[:sample_points]
    coords, sids = data.coords[idx], data.slice_ids[idx]
    up = np.random.default_rng(0).normal(size=len(idx)) * 1e-5
    t0 = time.perf_counter()
    inten, cnt = O.psf_render(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, 5, coords, sids,
                              ts.quats, ts.translations, psf.offsets, psf.weights, psf.through_dirs, threads)
    O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, 5, coords, sids, ts.quats,
                   ts.translations, psf.offsets, psf.weights, psf.through_dirs, up, threads)
    dt = time.perf_counter() - t0
    pairs = int(cnt.sum())
    return pairs / dt, pairs, dt, len(idx)


def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return
    import torch  # noqa: F401  (workload generator imports it)

    from oracle import oracle as O

    threads = os.cpu_count() or 1
    data, cloud, grids, psf, cfg = make_workload(args.config, 0)
    from paper_2603_00145_b200.core import uniform_lattice_field

    r = cfg.resolution_schedule[0][1]
    f = uniform_lattice_field(r)
    f.intensity_logits[:] = O.init_logits(data.coords, data.intensities, r)
    rng = np.random.default_rng(7)
    per_step = max(1024, args.cpu_sample_points)
    total_pairs, total_t = 0, 0.0
    for s in range(args.warmup + args.steps):
        idx = rng.choice(data.coords.shape[0], per_step, replace=False)
        coords, sids = data.coords[idx], data.slice_ids[idx]
        up = rng.normal(size=per_step) * 1e-5
        t0 = time.perf_counter()
        _, cnt = O.psf_render(f.positions, f.quaternions, f.log_scales, f.intensity_logits, r, 5, coords, sids,
                              data.transforms.quats, data.transforms.translations, psf.offsets, psf.weights,
                              psf.through_dirs, threads)
        O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, r, 5, coords, sids,
                       data.transforms.quats, data.transforms.translations, psf.offsets, psf.weights,
                       psf.through_dirs, up, threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            total_pairs += int(cnt.sum())
            total_t += dt
    v = total_pairs / total_t
    sample = (f"{per_step} batch points x {psf.ntaps} PSF taps per step (of 65,536 + 25,600), fwd+bwd incl. "
              f"activation/binning/epilogue, C2 field R={r}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * total_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, data, cfg, psf, np.asarray(grids[0].target).shape),
                   "cpu_threads": threads},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_ours(args):
    import torch

    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    group = None
    dist_on = world > 1 or args.force_dist
    if dist_on:
        import torch.distributed as tdist

        if not tdist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            tdist.init_process_group("nccl", rank=rank, world_size=world)
        group = tdist.group.WORLD
    from paper_2603_00145_b200 import _native as N
    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = make_workload(args.config, rank)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=not args.no_graph,
                 dist=group)
    # warm-up (eager first step, then graph capture + replays)
    for _ in range(max(args.warmup, 3)):
        tr.step(sync=True)
    # pre-generate the timed steps' indices on the host RNG, upload -> device-resident inputs
    steps_idx = []
    for _ in range(args.steps):
        idx = tr._next_batch()
        j = int(tr.rng.integers(len(tr.slice_grids)))
        all_idx, hw = tr.host_indices(idx, j)
        steps_idx.append(torch.from_numpy(all_idx).cuda())
    nb = cfg.batch_points
    B = tr._buffers(len(steps_idx[0]))
    B.pairs.zero_()
    sampler = ClockSampler(local)
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        tr.load_indices(steps_idx[k])
        if tr._graph is not None:
            tr._graph.replay()
        else:
            tr._body(B, nb, hw)
        tr.iteration += 1
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if dist_on:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    pairs_local = int(B.pairs.item())
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    pt = torch.tensor([pairs_local], dtype=torch.float64, device="cuda")
    if dist_on:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(pt)
    ms_max = float(t.item())
    pairs_total = float(pt.item())
    value = pairs_total / (ms_max / 1000.0)

    # --- the same steps with L2 flushed before each one (a 256 MB write, outside
    # the per-step event pairs): how much the L2-resident model state is worth ---
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    B.pairs.zero_()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        ev[k][0].record()
        tr.load_indices(steps_idx[k])
        if tr._graph is not None:
            tr._graph.replay()
        else:
            tr._body(B, nb, hw)
        ev[k][1].record()
        tr.iteration += 1
    torch.cuda.synchronize()
    msf = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device="cuda")
    pf = torch.tensor([int(B.pairs.item())], dtype=torch.float64, device="cuda")
    if dist_on:
        torch.distributed.all_reduce(msf, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(pf)
    del flush
    l2_flushed = {"ms_per_step": float(msf.item()) / args.steps, "value": float(pf.item()) / (float(msf.item()) / 1e3),
                  "method": "256 MB device write before every step, per-step CUDA events exclude it"}
    pool_bytes = sum(x.numel() * x.element_size() for x in (tr.src_coords, tr.src_sids, tr.src_tgt))

    # --- kernel-level timing (CUDA events around the pair kernels, eager, same stream) ---
    kt = kernel_times(tr, steps_idx[: min(5, len(steps_idx))], nb, hw)

    # --- end to end through the public API: Trainer.step() with host RNG batches (H2D) + loss D2H ---
    e2e_steps = max(30, args.steps)  # enough steps that the one-step pipeline fill/drain is amortised
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p_before = int(B.pairs.item())
    for _ in range(e2e_steps):  # host prep of step t+1 overlaps step t; indices up, losses down every step
        tr.step_pipelined()
    tr.flush()
    torch.cuda.synchronize()
    e2e_dt = time.perf_counter() - t0
    e2e_pairs = int(B.pairs.item()) - p_before
    e2e_t = torch.tensor([e2e_dt], dtype=torch.float64, device="cuda")
    e2e_p = torch.tensor([e2e_pairs], dtype=torch.float64, device="cuda")
    if dist_on:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(e2e_p)
    e2e_val = float(e2e_p.item()) / float(e2e_t.item())

    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    peaks = load_peaks()
    sms = N.lib().mg_device_sm_count()
    mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak = peak_fp32(sms, mhz)
    fwd_ms, bwd_ms, kpairs = kt["forward_ms"], kt["backward_ms"], kt["pairs_per_launch"]
    achieved_fwd = kpairs * FLOP_FWD / (fwd_ms / 1e3)
    achieved_bwd = kpairs * FLOP_BWD / (bwd_ms / 1e3)
    achieved_pair = kpairs * (FLOP_FWD + FLOP_BWD) / ((fwd_ms + bwd_ms) / 1e3)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("pair_kernels_dram_bytes")
        except Exception:
            traffic = None
    nlaunch = kt.get("launches_per_step")
    cpu = None
    if world == 1:  # the CPU baseline is an N = 1 figure (rank 0 alone at N > 1 would only add minutes)
        threads = os.cpu_count() or 1
        v, p, dt, npts = cpu_baseline(tr, data, psf, args.cpu_sample_points, threads)
        v1, p1, dt1, npts1 = cpu_baseline(tr, data, psf, max(1024, args.cpu_sample_points // 16), 1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{npts} batch points x {psf.ntaps} taps of one C2 step ({p} pairs, {dt:.1f} s), "
                         f"fwd+bwd incl. host epilogue",
               "value_1thread": v1, "sample_1thread": f"{npts1} batch points ({p1} pairs, {dt1:.1f} s)"}
    graph_used = tr._graph is not None
    tr.close()
    del tr
    torch.cuda.empty_cache()
    infer = None
    if not args.no_inference:
        try:
            infer = inference_c5()
        except Exception as exc:  # report, never fail the training bench
            infer = {"error": repr(exc)[:200]}
        torch.cuda.empty_cache()
    recon = None
    if not args.no_recon and rank == 0:
        try:
            recon = recon_desk64()
        except Exception as exc:
            recon = {"error": repr(exc)[:200]}
    bytes_h2d = int(steps_idx[0].numel() * 8)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "samples_per_s": world * float(steps_idx[0].numel()) * args.steps / (ms_max / 1000.0),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, data, cfg, psf, hw),
                   "global_batch": nb * world, "pairs_per_step": pairs_total / args.steps,
                   "parallelism": f"dp{world}", "l2": f"inputs larger than L2: every step gathers its batch at fresh random indices "
                   f"from the {pool_bytes / 2**20:.0f} MiB device sample pool (L2 126 MB); the model state "
                   f"(Gaussians + Adam moments) stays L2-resident across steps as in training. "
                   f"Also timed with L2 flushed before every step: see l2_flushed",
                   "cuda_graph": graph_used},
        "l2_flushed": l2_flushed,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": bytes_h2d, "d2h_bytes_per_step": 32 + 4,
                "path": "Trainer.step_pipelined(): host RNG batch -> pinned H2D -> graph replay -> async loss D2H, resolved one step later"},
        "roofline": {"bound": "fp32", "achieved": achieved_pair / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                     "frac": achieved_pair / peak, "traffic": traffic,
                     "peak_source": f"nominal 256 FLOP/clk/SM x {sms} SMs x {mhz:.0f} MHz (measured SM clock); "
                                    "MEASURED_PEAKS.json has no FP32 figure",
                     "kernels": {"forward": {"ms": fwd_ms, "tflops": achieved_fwd / 1e12,
                                             "frac": achieved_fwd / peak},
                                 "backward": {"ms": bwd_ms, "tflops": achieved_bwd / 1e12,
                                              "frac": achieved_bwd / peak},
                                 "pairs_per_launch": kpairs, "flop_per_pair": [FLOP_FWD, FLOP_BWD]}},
        "cpu_baseline": cpu,
        "inference": infer,
        "recon": recon,
        "clocks": clocks,
        "gpu_launches": (nlaunch * args.steps) if nlaunch else None,
        "gpu_launches_note": "library kernels per step (mg_launch_count over one eager step) x timed steps; "
                             "torch index_select/sum/fill plumbing kernels not counted",
    }
    print(json.dumps(out))
    if dist_on:
        torch.distributed.destroy_process_group()


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


def inference_c5(reps=3):
    """C5 (BASELINE.json configs[4]): sample a 512^3 node-inclusive volume over
    [-1, 1]^3 from a 2,000,376-Gaussian field (R = G = 126, r = 5).  Synthetic
    field per SURVEY §8(d): lattice positions + N(0, 0.1/R) jitter, identity +
    N(0, 0.1) quaternions, log-scales log(1/R) + N(0, 0.1), logits N(0, 1)."""
    import torch

    from paper_2603_00145_b200 import _native as N
    from paper_2603_00145_b200.core import lattice_node_positions
    from paper_2603_00145_b200.render import sample_volume_device
    from paper_2603_00145_b200.spatial import build_device

    R = 126
    n = R ** 3
    rng = np.random.default_rng(7)
    pos = lattice_node_positions(R) + rng.normal(0, 0.1 / R, (n, 3))
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    q += rng.normal(0, 0.1, (n, 4))
    ls = np.log(1.0 / R) + rng.normal(0, 0.1, (n, 3))
    lg = rng.normal(0, 1, n)
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
    return {"workload": "C5: 512^3 volume from 2,000,376 Gaussians (R=G=126, r=5), synthetic lattice field",
            "ms": ms, "voxels_per_s": 512 ** 3 / (ms / 1e3), "pairs_per_s": pairs / (ms / 1e3),
            "pairs": pairs, "roofline_frac_fp32": pairs * FLOP_FWD / (ms / 1e3) / peak}


def kernel_times(tr, idx_list, nb, hw):
    """Average device time of the forward and backward pair kernels, via CUDA
    events on the launching (current) stream, eager replays of timed batches."""
    import torch

    from paper_2603_00145_b200 import _native as N

    L = N.lib()
    fwd, bwd, upd, pairs = [], [], [], []
    orig_fwd, orig_bwd, orig_upd = L.mg_forward, L.mg_backward, L.mg_gauss_update

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

    B = tr._buffers(len(idx_list[0]))
    launches = []
    try:
        L.mg_forward, L.mg_backward, L.mg_gauss_update = Timed(orig_fwd, fwd), Timed(orig_bwd, bwd), Timed(orig_upd, upd)
        for ix in idx_list:
            tr.load_indices(ix)
            c0 = L.mg_launch_count()
            tr._body(B, nb, hw)
            launches.append(L.mg_launch_count() - c0)
            torch.cuda.synchronize()
            pairs.append(int(B.cnt.sum().item()))
    finally:
        L.mg_forward, L.mg_backward, L.mg_gauss_update = orig_fwd, orig_bwd, orig_upd
    torch.cuda.synchronize()
    f = float(np.mean([a.elapsed_time(b) for a, b in fwd]))
    b = float(np.mean([a.elapsed_time(c) for a, c in bwd]))
    u = float(np.mean([a.elapsed_time(c) for a, c in upd])) if upd else None
    return {"forward_ms": f, "backward_ms": b, "update_ms": u, "pairs_per_launch": float(np.mean(pairs)),
            "launches_per_step": int(max(launches))}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
