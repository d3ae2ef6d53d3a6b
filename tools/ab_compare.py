"""A/B of two builds of libbosrm.so on the same seeded workloads (development tool).

    BOS_LIBRARY=... python tools/ab_compare.py dump /tmp/a.npz
    BOS_LIBRARY=... python tools/ab_compare.py dump /tmp/b.npz
    python tools/ab_compare.py compare /tmp/a.npz /tmp/b.npz

`dump` demodulates C3 frames 1..F (M = 8, 11) and two C4 frames (M = 16, 24, 32) against
their reference frame and stores the phase maps; `compare` counts pixels whose wrapped
difference exceeds 1e-4 rad and checks up to 40 of them per case against the FP64 oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# (workload, M, flow frames, SNR dB override or None = the workload's own)
CASES = [("C3", 8, 20, None), ("C3", 11, 20, None), ("C4", 16, 2, None), ("C4", 24, 2, None), ("C4", 32, 2, None)]
if os.environ.get("AB_SNR_SET"):
    CASES = [("C3", 8, 10, 0.0), ("C3", 11, 10, 0.0), ("C3", 15, 4, 0.0), ("C3", 8, 10, 5.0), ("C3", 8, 10, 20.0),
             ("C3", 8, 10, 40.0), ("C1", 8, 0, None), ("C1", 9, 0, None), ("C4", 12, 2, 0.0), ("C4", 16, 2, 5.0)]


def stack_for(name, nframes, snr=None):
    from paper_1910_11872_b200 import synth
    w = synth.workload(name)
    s = "default" if snr is None else snr
    if nframes == 0:                                     # single-frame workloads: frame twice
        f = synth.make_frame(w, 0, snr_db=s)
        import torch
        return torch.stack([f, f])
    return synth.make_stack(w, frames=range(nframes + 1), snr_db=s)


def key(name, M, snr):
    return f"{name}_M{M}" + ("" if snr is None else f"_{snr:g}dB")


def dump(path):
    import torch
    from paper_1910_11872_b200 import bosrm
    out = {}
    for name, M, F, snr in CASES:
        st = stack_for(name, F, snr).to("cuda")
        ph, _, _ = bosrm.bos_rootmusic_demod_stack(st, M, ref_index=0)
        torch.cuda.synchronize()
        out[key(name, M, snr)] = ph[1:].cpu().numpy()
        del st, ph
    np.savez(path, **out)


def compare(pa, pb):
    from oracle import rootmusic as R
    a, b = np.load(pa), np.load(pb)
    for name, M, F, snr in CASES:
        k = key(name, M, snr)
        d = np.abs(R.wrap(a[k].astype(np.float64) - b[k]))
        bad = np.argwhere(np.nan_to_num(d, nan=10.0) > 1e-4)
        line = f"{k}: {d.size} px, {len(bad)} differ > 1e-4 rad"
        if len(bad):
            st = stack_for(name, F, snr).numpy()
            ea, eb = [], []
            for t, y, x in bad[:40]:
                o, _ = R.demod_stack(st[[0, t + 1]], M, pixels=(np.array([y]), np.array([x])), frame_indices=[1])
                ea.append(abs(R.wrap(a[k][t, y, x] - o[0][0])))
                eb.append(abs(R.wrap(b[k][t, y, x] - o[0][0])))
            line += (f"; vs oracle on {len(ea)}: A max {max(ea):.2e} (>{1e-2}: {sum(e > 1e-2 for e in ea)}), "
                     f"B max {max(eb):.2e} (>{1e-2}: {sum(e > 1e-2 for e in eb)})")
        print(line, flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    else:
        compare(sys.argv[2], sys.argv[3])
