"""C4 roofline study (BASELINE config 4): window_len sweep on 2048² diffusion frames, one B200.

For each M: device-resident stack of F frames (C4 generator: reference + flow frames at
t = 60 + 30k s, SNR 10 dB), warm-up, then CUDA-event time of `bos_rootmusic_demod` over the
stack (against the reference phase), the measured iteration counts, the algorithmic flop
model of bench.py and the FP32 roofline fraction.  Also a sampled parity check (1024 pixels
of one frame vs the FP64 oracle).  Prints a markdown table and one JSON line per M.

    python tools/sweep_window.py --sizes 8,9,11,12,15,16,17,20,24,28,32 --frames 8
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import rootmusic as R  # noqa: E402
from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8,9,11,12,15,16,17,20,24,28,32")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--parity-px", type=int, default=1024, help="sampled pixels of one frame checked vs the oracle")
    ap.add_argument("--variant", default="paper", choices=["paper", "fb", "fp64", "fb_fp64"],
                    help="row f4 variants (timing + parity vs the oracle of the same variant; no iteration counts)")
    ap.add_argument("--subarray", default="0",
                    help="row f4 spatial smoothing order m: an int (0 = none) or 'half' (m = M // 2, ≥ 3)")
    args = ap.parse_args()

    def sub_of(M_):
        if args.subarray == "half":
            return max(3, M_ // 2)
        return int(args.subarray)
    fb = args.variant != "paper" or args.subarray != "0"
    vbits = {"paper": 0, "fb": bosrm.VARIANT_FB, "fp64": bosrm.VARIANT_FP64,
             "fb_fp64": bosrm.VARIANT_FB | bosrm.VARIANT_FP64}[args.variant]
    ovar = "fb" if args.variant.startswith("fb") else "paper"

    def demod(frames_, M_, ref_=None, out_=None):
        if fb:
            return bosrm.bos_rootmusic_demod_variant(frames_, M_, variant=vbits, ref_phase=ref_,
                                                     out_phase=out_, subarray_len=sub_of(M_))[:2]
        return bosrm.bos_rootmusic_demod(frames_, M_, ref_phase=ref_, out_phase=out_)

    dev = torch.device("cuda", 0)
    w = synth.workload("C4", H=args.size, W=args.size)
    T = args.frames
    frames = synth.make_stack(w, frames=range(T), device=dev)
    plane = w.H * w.W
    peak = bench.B200_SMS * bench.FP32_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    rows = []
    print("| M | Mpixel/s | frames/s at 2048² | power its | Aberth sweeps y/x | kflop/px | TFLOP/s | frac of 74.45 | parity rms / max (rad) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for M in [int(x) for x in args.sizes.split(",")]:
        ref, _ = demod(frames[0:1], M)
        ref = ref[0].contiguous()
        out = torch.empty(T, w.H, w.W, dtype=torch.float32, device=dev)
        demod(frames, M, ref, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            demod(frames, M, ref, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        mpx = T * plane / (ms / 1e3) / 1e6
        if fb:
            kpi = ky = kx = float("nan")
            fpx = float("nan")
        else:
            cnt = bosrm.bos_rootmusic_iteration_counts(frames[1:2], M)
            npx = cnt["pixels"]
            kpi, ky, kx = cnt["power_its"] / npx, cnt["aberth_y"] / npx, cnt["aberth_x"] / npx
            fpx = bench.path_flops(M, kpi, ky, kx, T, w.H, w.W)
        tf = fpx * mpx * 1e6 / 1e12
        rng = np.random.default_rng(M)
        pix = (rng.integers(0, w.H, args.parity_px), rng.integers(0, w.W, args.parity_px))
        host = frames[[0, T - 1]].cpu().numpy()
        o, ofl = R.demod_stack(host, M, pixels=pix, frame_indices=[1], variant=ovar,
                               subarray_len=(sub_of(M) or None) if fb else None)
        g = out[T - 1].cpu().numpy()[pix]
        valid = (ofl[0] & R.PARITY_EXCLUDE_MASK) == 0
        e = R.wrap(g - o[0])[valid]
        rms, mx = float(math.sqrt(np.mean(e * e))), float(np.max(np.abs(e)))
        row = dict(M=M, variant=args.variant, subarray=sub_of(M), mpix_s=mpx, fps_2048=mpx / (plane / 1e6), power_its=kpi, aberth_y=ky, aberth_x=kx,
                   kflop_px=fpx / 1e3, tflops=tf, frac=tf / peak, parity_rms=rms, parity_max=mx,
                   kernel=bench.kernel_name(M, T, w.H, w.W) if not fb else "variant")
        rows.append(row)
        print(f"| {M} | {mpx:.1f} | {row['fps_2048']:.1f} | {kpi:.2f} | {ky:.2f}/{kx:.2f} | {fpx / 1e3:.1f} | "
              f"{tf:.1f} | {tf / peak:.3f} | {rms:.1e} / {mx:.1e} |", flush=True)
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
