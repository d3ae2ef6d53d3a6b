"""One warm-up + one profiled demod launch on C4 2048² frames (for per-M ncu studies).

    ncu --metrics ... -k regex:demod -s 1 -c 1 python tools/one_launch.py --M 20 --frames 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, required=True)
    ap.add_argument("--frames", type=int, default=1)
    args = ap.parse_args()
    w = synth.workload("C4")
    fr = synth.make_stack(w, frames=range(1, args.frames + 1), device=torch.device("cuda", 0))
    out = torch.empty(args.frames, w.H, w.W, dtype=torch.float32, device=fr.device)
    for _ in range(2):
        bosrm.bos_rootmusic_demod(fr, args.M, out_phase=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
