#!/usr/bin/env python
"""Benchmark: root-MUSIC demod throughput (Mpixel/s, frames/s at 1024²) on N B200s.

    python bench.py --gpus N --steps K --warmup W            # CUDA path (libbosrm.so)
    python bench.py --workload C5 --gpus N ...               # fixed 2048²×2000 stack, strong scaling
    python bench.py --impl reference --gpus N --steps K ...  # FP64 CPU oracle (rank 0 only)

Default workload (BASELINE.json configs[2]): C3 — a 1024×1024 time-lapse stack of
100 frames per rank (local frame 0 = the carrier-only reference, 99 diffusion flow frames),
window_len 8, model_order 3, SNR 10 dB, generated on the device before timing.  One step =
the whole hot path over the stack: demodulate the reference (raw α), then all 100 frames
against it (2 launches).  Weak scaling: every rank owns 99 distinct flow frames; value =
distinct output pixels of the job / max-over-ranks time.  This is also what the driver's
N = 1, 2, 4, 8 scaling run measures.

--workload C5 (configs[4]): ONE 2048²×2000 stack; rank r owns frames [⌊rT/G⌋, ⌊(r+1)T/G⌋)
(sharding.fixed_stack_indices) plus the reference; strong scaling, value = 2000·2048² / time.

At N = 1 the line also carries ``extra``: the paper's own operating points measured in the
same run — C2 512² pairs at 0/10/20 dB with M = 11 and M = 8, C3 at M = 15
(the experiment's L = 7), and the C5 stack on one GPU.
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
    p.add_argument("--workload", default="C3", choices=["C3", "C5"])
    p.add_argument("--frames", type=int, default=None, help="C3: frames per rank incl. the reference (100); "
                   "C5: frames of the whole stack (2000)")
    p.add_argument("--size", type=int, default=None, help="frame side (C3: 1024, C5: 2048)")
    p.add_argument("--no-extra", action="store_true", help="skip the N=1 extra operating points")
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


STRIP_ROWS = 16      # BOS_STRIP_ROWS: rows per strip work item on large launches (launch_strip)
STRIP_MIN_ROWS = 8   # BOS_STRIP_MIN_ROWS: launches that would get shorter strips run the row kernel
STRIP_SMALL_MIN_M = 17   # BOS_STRIP_SMALL_MIN_M: ... except the implicit kernel from this M


def strip_kind(M: int) -> int:
    """csrc/demod_strip.cuh strip_kind<M>(): 1 = R_y slid in registers, 2 = no R_y (implicit
    power iteration y = Γ_w(Γ_w^H u))."""
    return 1 if (M <= 10 or M in (12, 13)) else 2


def covariance_flops(M: int, strip_rows: int | None) -> float:
    """R_y = Γ_wΓ_w^H per pixel: 4M³ when formed in full (row / warp kernels); on the register
    strip kernel one full build per S-row strip and, for the other S−1 rows, only the new last
    row (M−1 complex MACs × M columns + the real diagonal entry: 8M(M−1) + 4M)."""
    full = 4.0 * M ** 3
    if not strip_rows:
        return full
    return (full + (strip_rows - 1) * (8.0 * M * (M - 1) + 4.0 * M)) / strip_rows


def flops_per_pixel(M: int, k_pi: float, k_aby: float, k_abx: float, strip_rows: int | None = None,
                    kind: int | None = None) -> float:
    """Algorithmic FP32 flops per pixel of the path, FMA = 2 flops.
    R_y and the power iteration, by kernel: explicit R_y (row / warp kernels, register strip
    kernel) — covariance (covariance_flops) + k_pi·(8M²+12M); implicit (kind 2, no R_y) — one
    pass for tr R_y and Σ R[i+1][i] 12M², then k_pi·(16M²+12M) (Γ_w^H u and Γ_w t: 2M² complex
    MACs).  Common: v_1 = Γ^H u_1 8M²+4M; two autocorrelation polynomials 8M(M−1); symmetric
    Aberth sweeps k·(n/2)·(25n+21) with n = 2M−2 (per tracked root: Horner for P and P′ 16n,
    n−1 reciprocal terms at 9 flops, mirror + update 30); selection 2·20(n/2); 2 Newton polish
    steps per axis 2·2·(16n+30); Eq.(15) 8M²+8M+20."""
    n = 2 * M - 2
    polish = 2 * 2 * (16.0 * n + 30.0)       # 2 Newton steps on the selected root, 2 axes
    if kind == 2:
        rpi = 12.0 * M * M + k_pi * (16.0 * M * M + 12.0 * M)
    else:
        rpi = covariance_flops(M, strip_rows) + k_pi * (8.0 * M * M + 12.0 * M)
    return (rpi + 8.0 * M * M + 4.0 * M
            + 8.0 * M * (M - 1) + (k_aby + k_abx) * (n / 2.0) * (25.0 * n + 21.0) + 20.0 * n
            + polish + 8.0 * M * M + 8.0 * M + 20.0)


def strip_rows_for(M: int, T: int = 100, H: int = 1024, W: int = 1024, sms: int = B200_SMS) -> int | None:
    """S the library's launcher picks for window M on a T×H×W launch (launch_strip: halve from
    BOS_STRIP_ROWS while fewer than 4 work items per resident warp, down to 2); None when the
    launch is too small for S ≥ BOS_STRIP_MIN_ROWS and runs the row / warp kernel."""
    warps_per_sm = (16 if M <= 8 else (12 if M <= 11 else 8)) if strip_kind(M) == 1 else (16 if M <= 11 else (12 if M <= 18 else 8))
    row_items = T * H * ((W + 31) // 32)
    S = STRIP_ROWS
    while S > 2 and row_items // S < 4 * warps_per_sm * sms:
        S //= 2
    any_size = strip_kind(M) == 2 and M >= STRIP_SMALL_MIN_M
    return S if (S >= STRIP_MIN_ROWS or any_size) else None


def path_flops(M: int, k_pi: float, k_aby: float, k_abx: float, T: int, H: int, W: int) -> float:
    """flops_per_pixel for the kernel the library runs on a T×H×W launch of window M."""
    S = strip_rows_for(M, T, H, W)
    if S is None:
        return flops_per_pixel(M, k_pi, k_aby, k_abx)
    kind = strip_kind(M)
    return flops_per_pixel(M, k_pi, k_aby, k_abx, strip_rows=S if kind == 1 else None, kind=kind)


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

    size = args.size or (2048 if args.workload == "C5" else 1024)
    w = synth.workload(args.workload, H=size, W=size, window_len=args.window_len)
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
    sample = (f"{n_px} random pixels x {F} flow frames of the {size}^2 {args.workload} stack per step, plus the "
              f"same pixels of the reference frame (W={w.window_len})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload} sample: {sample}", "H": size, "W": size,
                   "window_len": w.window_len, "model_order": 3},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


WIDE_MIN_M = 21   # first window on the warp-per-pixel kernel (BOS_WIDE_MIN_M, csrc/demod_wide.cuh)


def kernel_name(M: int, T: int = 100, H: int = 1024, W: int = 1024) -> str:
    if strip_rows_for(M, T, H, W):
        return f"bos::{'demod_strip_kernel' if strip_kind(M) == 1 else 'demod_strip_im_kernel'}<{M},false>"
    return f"bos::{'demod_kernel' if M < WIDE_MIN_M else 'demod_wide_kernel'}<{M},false,false>"


def measured_fp32_peak(dev_index: int):
    """FFMA / FFMA2 / MUFU.RCP peaks of this GPU from tools/microbench (built by build())."""
    exe = os.path.join(ROOT, "tools", "microbench")
    if not os.path.exists(exe):
        return None
    try:
        p = subprocess.run([exe, str(dev_index)], capture_output=True, text=True, timeout=120)
        return json.loads(p.stdout.strip().splitlines()[-1])
    except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
        return None


class StackTimer:
    """One step = the hot path over a resident stack: raw α (and flags) of the reference (local
    frame 0), then the T−1 flow frames against it (sharding.sharded_stack_step; 2 launches —
    the reference is demodulated once, as bos_rootmusic_demod_stack does).  Device times with
    CUDA events on the launching stream, barrier + synchronize around the region, max over
    ranks."""

    def __init__(self, frames, M, ref_mode, dev):
        from paper_1910_11872_b200 import bosrm
        T, H, W = frames.shape
        self.bosrm, self.frames, self.M, self.ref_mode, self.dev = bosrm, frames, M, ref_mode, dev
        self.out = torch.empty(T, H, W, dtype=torch.float32, device=dev)
        self.flags = torch.empty(T, H, W, dtype=torch.uint8, device=dev)
        self.ref = torch.empty(H, W, dtype=torch.float32, device=dev)
        self.stream = torch.cuda.current_stream(dev)

    def _raw(self, frame):
        H, W = frame.shape
        self.bosrm.bos_rootmusic_demod(frame.unsqueeze(0), self.M, out_phase=self.ref.view(1, H, W),
                                       flags=self.flags[:1])
        return self.ref

    def step(self, ev=None):
        from paper_1910_11872_b200 import sharding

        def demod_all(fr, r):
            # the flow frames (local 1…T−1) against φ_ref; the reference frame itself was
            # demodulated once by _raw (its own difference output ≡ 0 is not rewritten)
            if ev is not None:
                ev[0].record(self.stream)
            self.bosrm.bos_rootmusic_demod(fr[1:], self.M, ref_phase=r, out_phase=self.out[1:], flags=self.flags[1:])
            if ev is not None:
                ev[1].record(self.stream)

        sharding.sharded_stack_step(self.frames, demod_all, self._raw, self.ref_mode, self.ref)

    def run(self, steps, warmup, clocks=None):
        """→ (max-over-ranks ms for `steps` steps, max-over-ranks mean ms of the T-frame launch, clocks)"""
        from paper_1910_11872_b200 import sharding
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        if sharding.is_dist():
            dist.barrier()
        if clocks is not None:
            clocks.start()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if sharding.is_dist():
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(self.stream)
        for k in range(steps):
            self.step(kev[k])
        t1.record(self.stream)
        torch.cuda.synchronize()
        if sharding.is_dist():
            dist.barrier()
        ck = clocks.stop() if clocks is not None else None
        ms = sharding.max_over_ranks(t0.elapsed_time(t1), self.dev)
        kms = sharding.max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in kev), self.dev)
        return ms, kms, ck


def iteration_means(frames, M):
    from paper_1910_11872_b200 import bosrm
    cnt = bosrm.bos_rootmusic_iteration_counts(frames, M)
    npx = max(1, cnt["pixels"])
    return cnt["power_its"] / npx, cnt["aberth_y"] / npx, cnt["aberth_x"] / npx


def stack_api_ms(frames, M, steps, warmup):
    """Device time of `steps` bos_rootmusic_demod_stack calls on a resident stack (CUDA events,
    synchronize on both sides) — how a user demodulates a small stack such as a C2 pair."""
    from paper_1910_11872_b200 import bosrm
    T, H, W = frames.shape
    out = torch.empty(T, H, W, dtype=torch.float32, device=frames.device)
    ref = torch.empty(H, W, dtype=torch.float32, device=frames.device)
    fl = torch.empty(T, H, W, dtype=torch.uint8, device=frames.device)
    for _ in range(warmup):
        bosrm.bos_rootmusic_demod_stack(frames, M, ref_index=0, ref_phase_out=ref, out_phase=out, flags=fl)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        bosrm.bos_rootmusic_demod_stack(frames, M, ref_index=0, ref_phase_out=ref, out_phase=out, flags=fl)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def extra_points(args, dev):
    """N = 1 only: the paper's operating points, each timed like the main step (device-resident
    stack, reference + frames, CUDA events, 2 warm-ups).  Small stacks are repeated so each
    timed region lasts ≥ 50 ms."""
    from paper_1910_11872_b200 import synth
    res = {}
    c2 = []
    w2 = synth.workload("C2")
    for snr in (0.0, 10.0, 20.0):
        st = synth.make_stack(w2, device=dev, snr_db=snr)
        for M in (11, 8):
            ms = stack_api_ms(st, M, 50, 3)           # the pair through bos_rootmusic_demod_stack
            px = 2 * 512 * 512 * 50
            k = iteration_means(st[1:], M)
            c2.append({"snr_db": snr, "window_len": M, "mpix_s": px / (ms / 1e3) / 1e6,
                       "iters": {"power": k[0], "aberth_y": k[1], "aberth_x": k[2]},
                       "flops_per_px": path_flops(M, *k, 2, 512, 512)})
        del st
    res["c2_pair_512"] = {"what": "512^2 reference + flow pair (C2), per-step = bos_rootmusic_demod_stack of the pair "
                                  "(small stack: both frames raw in one launch, then the reference difference), 50 steps",
                          "points": c2}
    for snr in (0.0, 10.0, 20.0):
        r0 = next(p for p in c2 if p["snr_db"] == snr and p["window_len"] == 11)
        r10 = next(p for p in c2 if p["snr_db"] == 10.0 and p["window_len"] == 11)
        res["c2_pair_512"][f"m11_{int(snr)}db_vs_10db"] = r0["mpix_s"] / r10["mpix_s"]
    # C3 at the experiment's window (L = 7 → M = 15)
    w3 = synth.workload("C3", window_len=15)
    st = synth.make_stack(w3, device=dev)
    tm = StackTimer(st, 15, "recompute", dev)
    ms, kms, _ = tm.run(3, 2)
    k = iteration_means(st[1:5], 15)
    f = path_flops(15, *k, 100, 1024, 1024)
    res["c3_m15"] = {"mpix_s": 100 * 1024 * 1024 * 3 / (ms / 1e3) / 1e6, "kernel": kernel_name(15),
                     "frac_own_model": f * 99 * 1024 * 1024 / (kms / 1e3) / 1e12 / nominal_peak(),
                     "iters": {"power": k[0], "aberth_y": k[1], "aberth_x": k[2]}}
    del tm, st
    torch.cuda.empty_cache()
    # C5 on one GPU: the whole fixed 2048²×2000 stack, one step (≈ 8.4e9 pixels)
    w5 = synth.workload("C5")
    st = torch.empty(w5.T, w5.H, w5.W, dtype=torch.complex64, device=dev)
    synth.make_stack(w5, device=dev, out=st)
    tm = StackTimer(st, 8, "recompute", dev)
    ms, kms, _ = tm.run(1, 1)
    res["c5_n1"] = {"frames": w5.T, "H": w5.H, "W": w5.W, "window_len": 8, "step_ms": ms,
                    "mpix_s": w5.T * w5.H * w5.W / (ms / 1e3) / 1e6, "kernel_ms": kms}
    del tm, st
    torch.cuda.empty_cache()
    return res


def nominal_peak(sm_mhz: float | None = None) -> float:
    """FP32 FMA peak, TFLOP/s: 148 SM × 128 lanes × 2 flop × the max SM clock (MEASURED_PEAKS)."""
    f = sm_mhz if sm_mhz is not None else float(peaks().get("sm_max_mhz", 1965.0))
    return B200_SMS * FP32_LANES_PER_SM * 2 * f * 1e6 / 1e12


def run_cuda(args, world, rank, local):
    from paper_1910_11872_b200 import bosrm, sharding, synth

    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl cuda needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    bosrm.lib()
    M = args.window_len
    c5 = args.workload == "C5"
    size = args.size or (2048 if c5 else 1024)
    H = W = size
    plane = H * W
    if c5:
        T_job = args.frames or 2000
        w = synth.workload("C5", H=H, W=W, window_len=M, T=T_job)
        gidx = sharding.fixed_stack_indices(rank, world, T_job)
        out_frames = T_job
        scaling = "strong"
    else:
        T_rank = args.frames or 100
        w = synth.workload("C3", H=H, W=W, window_len=M)
        gidx = sharding.rank_frame_indices(rank, world, T_rank)
        out_frames = sharding.distinct_output_frames(world, T_rank)
        scaling = "weak"
    T = len(gidx)
    frames = torch.empty(T, H, W, dtype=torch.complex64, device=dev)
    synth.make_stack(w, frames=gidx, device=dev, out=frames)
    torch.cuda.synchronize()

    # iteration counts for the algorithmic flop model (outside the timed region)
    k_pi, k_aby, k_abx = iteration_means(frames[1:min(T, 5)], M)
    mb = measured_fp32_peak(dev.index) if rank == 0 else None

    tm = StackTimer(frames, M, args.ref_mode, dev)
    elapsed_ms, kern_ms, clocks = tm.run(args.steps, args.warmup, ClockSampler(dev.index))
    out, flags = tm.out, tm.flags

    units = out_frames * plane * args.steps
    value = units / (elapsed_ms / 1e3) / 1e6
    ms_per_step = elapsed_ms / args.steps

    # roofline of the dominant kernel (the T-frame demod launch; the ref launch is 1/T of it)
    f_px = path_flops(M, k_pi, k_aby, k_abx, T - 1, H, W)
    achieved = f_px * (T - 1) * plane / (kern_ms / 1e3) / 1e12     # the timed launch: the T−1 flow frames
    sm_max = float(peaks().get("sm_max_mhz", 1965.0))
    peak = nominal_peak(sm_max)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        if int(tr.get("window_len", -1)) == M:
            traffic = tr["dram_bytes_per_pixel"] * (T - 1) * plane   # bytes per flow-frame launch (ncu capture)
    except (OSError, ValueError, KeyError):
        traffic = None
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read+write, profiles/)",
                "kernel": kernel_name(M, T, H, W), "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                "flops_per_px": f_px, "iters": {"power": k_pi, "aberth_y": k_aby, "aberth_x": k_abx},
                "peak_basis": f"nominal FP32 FMA (the contract): {B200_SMS} SM x {FP32_LANES_PER_SM} lanes x 2 x "
                              f"{sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                "hbm_gbs": ((T - 1) * plane * 13 + plane * 4) / (kern_ms / 1e3) / 1e9}
    if mb and mb.get("ffma_tflops"):
        roofline["peak_measured_ffma"] = mb["ffma_tflops"]
        roofline["frac_vs_measured_ffma"] = achieved / mb["ffma_tflops"]
        roofline["microbench"] = mb
    if clocks and clocks.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = achieved / nominal_peak(clocks["sm_mhz"])

    # e2e: the same step through the C-ABI host-buffer entry point (H2D/D2H in the region)
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(1, min(args.steps, 10 if not c5 else 1))
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
        stream = torch.cuda.current_stream(dev)
        a.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = sharding.max_over_ranks(a.elapsed_time(b), dev)
        e2e = {"value": out_frames * plane * e2e_steps / (e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": T * plane * 8, "d2h_bytes_per_step": T * plane * 5,
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
        sample = (f"{args.cpu_sample_px} random pixels x {F} flow frames of this {args.workload} stack, plus the same "
                  f"pixels of the reference frame ({dt:.1f} s wall)")
        cpu_baseline = {"value": cpu_val, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample}
        # parity of the timed GPU output at the same pixels (north_star tolerance)
        from oracle import rootmusic as R
        g = out[1:F + 1].cpu().numpy()[:, pix[0], pix[1]]
        valid = (ofl & R.PARITY_EXCLUDE_MASK) == 0
        e = R.wrap(g - o)[valid]
        gpu_nan = int(np.sum(~np.isfinite(e)))          # NaN on an oracle-valid pixel is a failure
        ef = e[np.isfinite(e)]
        gfl = flags[1:F + 1].cpu().numpy()[:, pix[0], pix[1]]
        gpu_only = ((gfl & R.PARITY_EXCLUDE_MASK) != 0) & valid     # flagged by the GPU, not the oracle
        parity = {"rms": float(math.sqrt(np.mean(ef * ef))) if ef.size else None,
                  "max": float(np.max(np.abs(ef))) if ef.size else None, "n": int(e.size), "gpu_nan": gpu_nan,
                  "excluded_frac": float(1 - valid.mean()), "gpu_only_flagged_frac": float(gpu_only.mean()),
                  "tol": {"rms": 1e-3, "max": 1e-2}}

    del tm, frames, out, flags
    torch.cuda.empty_cache()
    extra = None
    if rank == 0 and world == 1 and not args.no_extra and not c5:
        extra = extra_points(args, dev)

    if rank == 0:
        if c5:
            wl = (f"C5: one {H}x{W} stack of {out_frames} frames (frame 0 = carrier-only reference, diffusion flow "
                  f"frames), frames [floor(rT/G), floor((r+1)T/G)) + the reference on rank r, window_len {M}, "
                  f"model_order 3, SNR 10 dB")
        else:
            wl = (f"C3: {H}x{W} time-lapse stack, {T} frames/rank (reference + {T - 1} diffusion flow frames), "
                  f"window_len {M}, model_order 3, SNR 10 dB")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "frames_per_s_1024": value / 1.048576,
            "config": {"workload": wl, "H": H, "W": W, "frames_per_rank": T, "window_len": M, "model_order": 3,
                       "ref_mode": args.ref_mode, "distinct_output_frames": out_frames,
                       "l2": f"inputs {T * plane * 8 / 2**20:.0f} MiB/rank > 126 MB L2 (no flush needed)"},
            "gpu_launches": 2 * args.steps,
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e, "clocks": clocks, "parity": parity,
            "extra": extra,
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
