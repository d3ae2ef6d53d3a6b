"""Worst-pixel dump for a demod variant on a C4 frame: GPU (FB or paper) vs the FP64 oracle
at sampled pixels, with the oracle's eigen-gap, selection margin and flags.

    python tools/debug_variant.py --M 32 --variant fb --n 4096
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rootmusic as R  # noqa: E402
from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--variant", default="fb")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--frame", type=int, default=3)
    ap.add_argument("--workload", default="C4", help="C4, C2 (flow frame, --snr) or ragged (test frame)")
    ap.add_argument("--snr", type=float, default=10.0)
    args = ap.parse_args()
    if args.workload == "ragged":
        M = args.M
        H, W = (37, 45) if M < 19 else (M + 6, 75)
        w = synth.workload("C3", H=H, W=W, seed=M)
        fr = synth.make_frame(w, 5, snr_db=10.0)[None]
    elif args.workload == "C2":
        w = synth.workload("C2")
        fr = synth.make_stack(w, snr_db=args.snr)[1:2]
    else:
        w = synth.workload("C4")
        fr = synth.make_stack(w, frames=[args.frame])
    v = bosrm.VARIANT_FB if args.variant == "fb" else bosrm.VARIANT_PAPER
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_variant(fr.to("cuda"), args.M, variant=v, flags=True, omega=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    if args.workload == "ragged":
        yy, xx = np.meshgrid(np.arange(w.H), np.arange(w.W), indexing="ij")
        py, px = yy.ravel(), xx.ravel()
    else:
        py, px = rng.integers(0, w.H, args.n), rng.integers(0, w.W, args.n)
    win, _ = R.extract_windows(fr[0].numpy(), py, px, args.M)
    r = R.estimate_windows(win, args.variant)
    g = out[0].cpu().numpy()[py, px]
    gfl = fl[0].cpu().numpy()[py, px]
    gwx, gwy = wx[0].cpu().numpy()[py, px], wy[0].cpu().numpy()[py, px]
    e = np.abs(R.wrap(g - r["alpha"]))
    ok = (r["flags"] & R.PARITY_EXCLUDE_MASK) == 0
    e[~ok] = -1
    gap = (r["S"][:, 0] / r["S"][:, 1]) ** 2
    if args.variant == "fb":
        _, _, _, Sx = R.fb_subspaces(win)
        gap = np.minimum(gap, (Sx[:, 0] / Sx[:, 1]) ** 2)
    print(f"M={args.M} variant={args.variant} workload={args.workload} n={py.size} rms={np.sqrt(np.mean(e[ok] ** 2)):.2e} max={e.max():.2e}")
    for i in np.argsort(-e)[:12]:
        print(f"({py[i]},{px[i]}) err={e[i]:.3e} gap={gap[i]:.3f} margin={r['margin'][i]:.2e} "
              f"oflag={r['flags'][i]} gflag={gfl[i]} wx {gwx[i]:+.5f}/{r['omega_x'][i]:+.5f} "
              f"wy {gwy[i]:+.5f}/{r['omega_y'][i]:+.5f}")


if __name__ == "__main__":
    main()
