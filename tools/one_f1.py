"""Two bos_analytic_signal calls on 16 C3 8-bit 1024² frames (for ncu launch lists /
captures of the row-f1 kernels).

    ncu --set full -k regex:f1_rows_inv -s 2 -c 1 python tools/one_f1.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def main():
    w = synth.workload("C3")
    fr = torch.stack([synth.make_intensity_frame(w, t) for t in range(16)]).cuda()
    for _ in range(2):
        bosrm.bos_analytic_signal(fr, synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
