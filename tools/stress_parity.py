"""Randomised GPU-vs-oracle parity stress (development tool): random window sizes, SNRs,
seeds, frame sizes and phase workloads; reports the worst wrapped error over oracle-unflagged
pixels per case and every case that breaks the north_star bar (RMS 1e-3, max 1e-2 rad).

    python tools/stress_parity.py --cases 200 --seed 1
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rootmusic as R  # noqa: E402
from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def draw_cases(seed, n, min_m=3, max_m=32):
    """The random case sequence of a seed: dicts with M, H, W, snr, workload, t, wseed (the
    default M range 3…32 reproduces the sequences quoted in DESIGN.md)."""
    rng = np.random.default_rng(seed)
    for c in range(n):
        M = int(rng.integers(min_m, max_m + 1))
        H = int(rng.integers(max(M, 8), 96))
        W = int(rng.integers(max(M, 8), 120))
        snr = float(rng.choice([-5.0, 0.0, 5.0, 10.0, 20.0, 40.0, np.inf]))
        wl = str(rng.choice(["C2", "C3", "C1"]))
        wseed = int(rng.integers(0, 1 << 30))
        t = int(rng.integers(1, 5)) if wl != "C1" else 0
        yield dict(case=c, M=M, H=H, W=W, snr=snr, workload=wl, t=t, wseed=wseed)


def run_case(k):
    """GPU vs oracle on one case; returns (max, rms, nan count, excluded fraction)."""
    w = synth.workload(k["workload"], H=k["H"], W=k["W"], seed=k["wseed"])
    f = synth.make_frame(w, k["t"], snr_db=None if k["snr"] == np.inf else k["snr"])
    var = k.get("variant", "paper")
    if var == "paper":
        g, _ = bosrm.bos_rootmusic_demod(f.to("cuda"), k["M"])
        o, ofl = R.demod_frame(f.numpy(), k["M"])
    else:
        fb = var in ("fb", "ss_fb")
        m = k.get("subarray", 0) if var.startswith("ss") else 0
        g, _, _, _ = bosrm.bos_rootmusic_demod_variant(
            f.to("cuda"), k["M"], variant=bosrm.VARIANT_FB if fb else bosrm.VARIANT_PAPER, subarray_len=m)
        o, ofl = R.demod_frame(f.numpy(), k["M"], variant="fb" if fb else "paper", subarray_len=m or None)
    torch.cuda.synchronize()
    valid = (ofl & R.PARITY_EXCLUDE_MASK) == 0
    e = np.abs(R.wrap(g[0].cpu().numpy().astype(np.float64) - o))[valid]
    nan = int(np.sum(~np.isfinite(e)))
    e = e[np.isfinite(e)]
    mx = float(e.max()) if e.size else 0.0
    rms = float(math.sqrt(np.mean(e * e))) if e.size else 0.0
    return mx, rms, nan, float(1 - valid.mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--budget-s", type=float, default=600.0)
    ap.add_argument("--variant", default="paper", choices=["paper", "fb", "ss", "ss_fb"])
    ap.add_argument("--subarray", type=int, default=3, help="spatial-smoothing subarray m (ss variants)")
    ap.add_argument("--min-m", type=int, default=3)
    ap.add_argument("--max-m", type=int, default=32)
    args = ap.parse_args()
    bad, worst, t0, c, worst_case = [], 0.0, time.time(), -1, None
    for k in draw_cases(args.seed, args.cases, args.min_m, args.max_m):
        if time.time() - t0 > args.budget_s:
            break
        c = k["case"]
        k = dict(k, variant=args.variant, subarray=args.subarray)
        if args.variant.startswith("ss") and k["M"] <= args.subarray:
            continue
        mx, rms, nan, exc = run_case(k)
        if mx > worst:
            worst, worst_case = mx, dict(M=k["M"], snr=k["snr"], H=k["H"], W=k["W"], workload=k["workload"])
        if nan or mx > 1e-2 or rms > 1e-3:
            bad.append(dict(k, max=mx, rms=rms, nan=nan, excluded=exc))
    print(f"cases run: {c + 1}, failures: {len(bad)}, worst max error {worst:.2e} rad"
          f" (kernel choice BOS_THREAD_KERNEL={os.environ.get('BOS_THREAD_KERNEL', 'auto')})")
    print(f"worst case: {worst_case}")
    for b in bad:
        print(b)


if __name__ == "__main__":
    main()
