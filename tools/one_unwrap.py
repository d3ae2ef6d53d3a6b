"""One warm-up + one bos_unwrap call on T 1024² demodulated C3 frames (for ncu launch lists).

    ncu --metrics gpu__time_duration.sum -k regex:'^(?!.*elementwise)' python tools/one_unwrap.py --frames 100
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
    ap.add_argument("--frames", type=int, default=100)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = synth.workload("C3")
    st = synth.make_stack(w, frames=range(a.frames), device=dev)
    ph, _, _ = bosrm.bos_rootmusic_demod_stack(st, 8, ref_index=0)
    del st
    for _ in range(2):
        bosrm.bos_unwrap(ph)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
