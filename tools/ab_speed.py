"""Throughput + iteration counts of one libbosrm.so build (BOS_LIBRARY=…) on fixed seeded stacks
(development A/B tool).  Cases: C3 1024² frames at 10 dB and 0 dB, window lengths from --ms.
Each case: a device-resident stack of --frames flow frames, one warm-up launch, then the mean
CUDA-event time of --reps launches against a reference phase.  Prints one JSON line per case.

    BOS_LIBRARY=abl/libbosrm_x.so python tools/ab_speed.py --ms 8,11,15 --snrs 10,0 --tag x
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1910_11872_b200 import bosrm, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="8,11,15")
    ap.add_argument("--snrs", default="10,0")
    ap.add_argument("--frames", type=int, default=16)
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default=os.environ.get("BOS_LIBRARY", "default"))
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--variant", default="paper", choices=["paper", "fb"])
    a = ap.parse_args()
    dev = torch.device("cuda")
    bosrm.lib()
    for snr in [float(s) for s in a.snrs.split(",")]:
        w = synth.workload(a.workload, H=a.size, W=a.size)
        st = synth.make_stack(w, frames=range(a.frames + 1), device=dev, snr_db=snr)
        for M in [int(m) for m in a.ms.split(",")]:
            ref = bosrm.bos_rootmusic_demod(st[:1], M)[0][0]
            fr = st[1:]
            out = torch.empty(fr.shape, dtype=torch.float32, device=dev)
            if a.variant == "fb":
                def run():
                    bosrm.bos_rootmusic_demod_variant(fr, M, variant=bosrm.VARIANT_FB, ref_phase=ref, out_phase=out)
            else:
                def run():
                    bosrm.bos_rootmusic_demod(fr, M, ref_phase=ref, out_phase=out)
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            c = bosrm.bos_rootmusic_iteration_counts(fr[:4], M, ref_phase=ref) if a.variant == "paper" else \
                dict(pixels=1, power_its=0, aberth_y=0, aberth_x=0)
            n = max(1, c["pixels"])
            print(json.dumps({"tag": a.tag, "variant": a.variant, "M": M, "snr": snr, "mpix_s": round(fr.numel() / ms / 1e3, 1),
                              "ms": round(ms, 3), "power": round(c["power_its"] / n, 3),
                              "aby": round(c["aberth_y"] / n, 3), "abx": round(c["aberth_x"] / n, 3)}), flush=True)
            del out
        del st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
