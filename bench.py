#!/usr/bin/env python
"""Benchmark: root-MUSIC demod throughput (Mpixel/s, frames/s at 1024²) on N B200s.

    python bench.py --gpus N --steps K --warmup W            # CUDA path (libbosrm.so)
    python bench.py --impl reference --gpus N --steps K ...  # FP64 CPU oracle (rank 0 only)

Workload (BASELINE.json configs[2]): C3 — a 1024×1024 time-lapse stack of 100
frames per rank (local frame 0 = the carrier-only reference, 99 diffusion flow frames),
window_len 8, model_order 3, SNR 10 dB, generated on the device before timing.  One step =
the whole hot path over the stack: demodulate the reference (raw α), then all 100 frames
against it (bos_rootmusic_demod_stack: 2 launches).  Weak scaling: every rank owns 99
distinct flow frames; value = distinct output pixels of the job / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "root-MUSIC demod Mpixel/s (frames/s at 1024²) at 1/2/4/8 B200 vs CPU oracle"
UNIT = "Mpixel/s"
FP32_LANES_PER_SM = 128          # FP32 FMA lanes per SM (Blackwell SM: 4 SMSP × 32)
B200_SMS = 148


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    p.add_argument("--frames", type=int, default=100, help="frames per rank (incl. the reference)")
    p.add_argument("--size", type=int, default=1024)
    p.add_argument("--window-len", type=int, default=8)
    p.add_argument("--ref-mode", default="recompute", choices=["recompute", "broadcast"])
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--chunk-frames", type=int, default=5)   # e2e pipeline chunk: 4 → 2589, 5 → 2624, 10 → 2547, 20 → 2298 Mpixel/s
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-px", type=int, default=8192)
    p.add_argument("--cpu-sample-frames", type=int, default=8)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def flops_per_pixel(M: int, k_pi: float, k_aby: float, k_abx: float) -> float:
    """Algorithmic FP32 flops per pixel of the path, FMA = 2 flops:
    covariance 4M³; power iteration k_pi·(8M²+12M); v_1 = Γ^H u_1 8M²+4M; two
    autocorrelation polynomials 8M(M−1); symmetric Aberth sweeps k·(n/2)·(25n+21) with
    n = 2M−2 (per tracked root: Horner for P and P′ 16n, n−1 reciprocal terms at 9 flops,
    mirror + update 30); selection 2·20(n/2); 2 Newton polish steps per axis 2·2·(16n+30);
    Eq.(15) 8M²+8M+20."""
    n = 2 * M - 2
    polish = 2 * 2 * (16.0 * n + 30.0)       # 2 Newton steps on the selected root, 2 axes
    return (4.0 * M ** 3 + k_pi * (8.0 * M * M + 12.0 * M) + 8.0 * M * M + 4.0 * M
            + 8.0 * M * (M - 1) + (k_aby + k_abx) * (n / 2.0) * (25.0 * n + 21.0) + 20.0 * n
            + polish + 8.0 * M * M + 8.0 * M + 20.0)


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nme, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nme)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # BOS_DIST_BACKEND=gloo: functional check of the N>1 code path on a single-GPU box (ranks
        # share the device; never a measurement)
        backend = os.environ.get("BOS_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def oracle_sample(host_frames: np.ndarray, M: int, n_px: int, seed: int = 0):
    """The FP64 oracle as it stands on a bounded sample: n_px random pixels of every host
    frame (index 0 = reference).  Returns (outputs [F-1,n_px], flags, pixels, seconds, threads)."""
    from oracle import rootmusic as R

    H, W = host_frames.shape[1:]
    rng = np.random.default_rng(seed)
    pix = (rng.integers(0, H, n_px), rng.integers(0, W, n_px))
    threads = R.default_threads()
    t0 = time.perf_counter()
    out, fl = R.demod_stack(host_frames, M, ref_index=0, pixels=pix,
                            frame_indices=list(range(1, host_frames.shape[0])), threads=threads)
    dt = time.perf_counter() - t0
    return out, fl, pix, dt, threads


def run_reference(args, world, rank):
    """--impl reference: the oracle on rank 0 (other ranks exit without work)."""
    if rank != 0:
        return
    from paper_1910_11872_b200 import synth

    w = synth.workload("C3", H=args.size, W=args.size, window_len=args.window_len)
    F = args.cpu_sample_frames
    n_px = max(256, args.cpu_sample_px)
    frames = synth.make_stack(w, frames=[0] + list(range(1, F + 1))).numpy()
    times = []
    threads = 1
    for i in range(args.warmup + args.steps):
        _, _, _, dt, threads = oracle_sample(frames, w.window_len, n_px, seed=i)
        if i >= args.warmup:
            times.append(dt)
    per_step = statistics.mean(times)
    outputs = n_px * F
    value = outputs / per_step / 1e6
    sample = (f"{n_px} random pixels x {F} flow frames of the {args.size}^2 C3 stack per step, plus the same "
              f"pixels of the reference frame (W={w.window_len})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C3 sample: {sample}", "H": args.size, "W": args.size,
                   "window_len": w.window_len, "model_order": 3},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_cuda(args, world, rank, local):
    from paper_1910_11872_b200 import bosrm, sharding, synth

    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl cuda needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    bosrm.lib()
    M = args.window_len
    T = args.frames
    w = synth.workload("C3", H=args.size, W=args.size, window_len=M)
    H = W = args.size
    plane = H * W
    gidx = sharding.rank_frame_indices(rank, world, T)
    frames = torch.empty(T, H, W, dtype=torch.complex64, device=dev)
    synth.make_stack(w, frames=gidx, device=dev, out=frames)
    out = torch.empty(T, H, W, dtype=torch.float32, device=dev)
    flags = torch.empty(T, H, W, dtype=torch.uint8, device=dev)
    ref = torch.empty(H, W, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    k_start = torch.cuda.Event(enable_timing=True)
    k_end = torch.cuda.Event(enable_timing=True)
    kernel_ms = []

    def demod_raw(frame):
        bosrm.bos_rootmusic_demod(frame.unsqueeze(0), M, out_phase=ref.view(1, H, W))
        return ref

    def demod_all(fr, r, timed=False):
        if timed:
            k_start.record(stream)
        bosrm.bos_rootmusic_demod(fr, M, ref_phase=r, out_phase=out, flags=flags)
        if timed:
            k_end.record(stream)

    def step(timed=False):
        sharding.sharded_stack_step(frames, lambda fr, r: demod_all(fr, r, timed), demod_raw, args.ref_mode, ref)

    # iteration counts for the algorithmic flop model (outside the timed region)
    cnt = bosrm.bos_rootmusic_iteration_counts(frames[1:min(T, 5)], M)
    npx = max(1, cnt["pixels"])
    k_pi, k_aby, k_abx = cnt["power_its"] / npx, cnt["aberth_y"] / npx, cnt["aberth_x"] / npx
    del cnt

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if sharding.is_dist():
        dist.barrier()
    sampler = ClockSampler(dev.index)
    sampler.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if sharding.is_dist():
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for _ in range(args.steps):
        step(timed=True)
        kernel_ms.append((k_start, k_end))
        k_start = torch.cuda.Event(enable_timing=True)
        k_end = torch.cuda.Event(enable_timing=True)
    t_end.record(stream)
    torch.cuda.synchronize()
    if sharding.is_dist():
        dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern = [a.elapsed_time(b) for a, b in kernel_ms]
    elapsed_ms = sharding.max_over_ranks(elapsed_ms, dev)
    kern_ms = sharding.max_over_ranks(statistics.mean(kern), dev)

    out_frames = sharding.distinct_output_frames(world, T)
    units = out_frames * plane * args.steps
    value = units / (elapsed_ms / 1e3) / 1e6
    ms_per_step = elapsed_ms / args.steps

    # roofline of the dominant kernel (the T-frame demod launch; ref launch is 1/T of it)
    P = peaks()
    f_px = flops_per_pixel(M, k_pi, k_aby, k_abx)
    achieved = f_px * T * plane / (kern_ms / 1e3) / 1e12
    sm_max = float(P.get("sm_max_mhz", 1965.0))
    peak = B200_SMS * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        if int(tr.get("window_len", -1)) == M:
            traffic = tr["dram_bytes_per_pixel"] * T * plane   # bytes per stack launch (ncu capture)
    except (OSError, ValueError, KeyError):
        traffic = None
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read+write, profiles/)", "kernel": f"bos::{'demod_kernel' if M <= 18 else 'demod_wide_kernel'}<{M},false,false>", "kernel_ms": kern_ms,
                "kernel_share_of_step": kern_ms / ms_per_step,
                "flops_per_px": f_px, "iters": {"power": k_pi, "aberth_y": k_aby, "aberth_x": k_abx},
                "peak_basis": f"FP32 FMA: {B200_SMS} SM x {FP32_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz",
                "hbm_gbs": (T * plane * 13 + plane * 8) / (kern_ms / 1e3) / 1e9}
    if clocks and clocks.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = achieved / (B200_SMS * FP32_LANES_PER_SM * 2 * clocks["sm_mhz"] / 1e6)

    # e2e: the same step through the C-ABI host-buffer entry point (H2D/D2H in the region)
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 5))
    if e2e_steps > 0:
        h_frames = frames.cpu().pin_memory()
        h_out = torch.empty(T, H, W, dtype=torch.float32).pin_memory()
        h_flags = torch.empty(T, H, W, dtype=torch.uint8).pin_memory()
        ws = torch.empty(bosrm.bos_rootmusic_host_workspace_bytes(H, W, args.chunk_frames, True),
                         dtype=torch.uint8, device=dev)

        def e2e_step():
            bosrm.bos_rootmusic_demod_stack_host(h_frames, M, ref_index=0, h_out_phase=h_out, h_flags=h_flags,
                                                 workspace=ws, chunk_frames=args.chunk_frames)

        e2e_step()
        torch.cuda.synchronize()
        if sharding.is_dist():
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = sharding.max_over_ranks(a.elapsed_time(b), dev)
        e2e = {"value": out_frames * plane * e2e_steps / (e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": (T + 1) * plane * 8, "d2h_bytes_per_step": T * plane * 5,
               "steps": e2e_steps, "chunk_frames": args.chunk_frames,
               "api": "bos_rootmusic_demod_stack_host (pinned host buffers)"}
        # consistency: the host path produced the device path's bytes
        e2e["matches_device"] = bool(torch.equal(h_out[: min(T, 4)], out[: min(T, 4)].cpu()))
        del h_frames, h_out, h_flags, ws

    cpu_baseline = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        F = min(args.cpu_sample_frames, T - 1)
        sel = [0] + list(range(1, F + 1))
        host = frames[sel].cpu().numpy()
        o, ofl, pix, dt, threads = oracle_sample(host, M, args.cpu_sample_px, seed=1)
        n_out = args.cpu_sample_px * F
        cpu_val = n_out / dt / 1e6
        sample = (f"{args.cpu_sample_px} random pixels x {F} flow frames of this C3 stack, plus the same pixels of "
                  f"the reference frame ({dt:.1f} s wall)")
        cpu_baseline = {"value": cpu_val, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample}
        # parity of the timed GPU output at the same pixels (north_star tolerance)
        from oracle import rootmusic as R
        g = out[1:F + 1].cpu().numpy()[:, pix[0], pix[1]]
        valid = (ofl & R.PARITY_EXCLUDE_MASK) == 0
        e = R.wrap(g - o)[valid]
        e = e[np.isfinite(e)]
        gfl = flags[1:F + 1].cpu().numpy()[:, pix[0], pix[1]]
        gpu_only = ((gfl & R.PARITY_EXCLUDE_MASK) != 0) & valid     # flagged by the GPU, not the oracle
        parity = {"rms": float(math.sqrt(np.mean(e * e))), "max": float(np.max(np.abs(e))), "n": int(e.size),
                  "excluded_frac": float(1 - valid.mean()), "gpu_only_flagged_frac": float(gpu_only.mean()),
                  "tol": {"rms": 1e-3, "max": 1e-2}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "frames_per_s_1024": value / 1.048576 * (1024 * 1024 / plane) if plane else None,
            "config": {"workload": f"C3: {H}x{W} time-lapse stack, {T} frames/rank (reference + {T - 1} diffusion "
                                   f"flow frames), window_len {M}, model_order 3, SNR 10 dB",
                       "H": H, "W": W, "frames_per_rank": T, "window_len": M, "model_order": 3,
                       "ref_mode": args.ref_mode, "distinct_output_frames": out_frames,
                       "l2": f"inputs {T * plane * 8 / 2**20:.0f} MiB/rank > 126 MB L2 (no flush needed)"},
            "gpu_launches": 2 * args.steps,
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e, "clocks": clocks, "parity": parity,
        }
        if cpu_baseline:
            line["speedup_vs_cpu_oracle"] = value / cpu_baseline["value"]
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = init_dist()
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_cuda(args, world, rank, local)
    finally:
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
