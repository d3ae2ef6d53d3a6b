"""Small invocation of every entry point and kernel family, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck — one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py

Covers: the thread-per-pixel kernel (R_y in registers: M = 3, 8, 11, 15, 16; in shared-memory
slices: M = 17, 20; cp.async double buffer at M ≤ 15), the warp-per-pixel kernel (M = 21, 24,
32), the FB variant on both kernels, spatial smoothing (m = 3 Ferrari, m = 5), the FP64 path,
the stack / host-pipeline entry points, f1 (analytic signal, per-call and planned), f2
(unwrap) and f3 (index gradient, vertical profile)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1910_11872_b200 import bosrm, synth  # noqa: E402

dev = "cuda"
w = synth.workload("C3", H=37, W=70)
st = synth.make_stack(w, frames=[0, 3, 9], device=dev)
Ms = [int(m) for m in os.environ.get("BOS_SAN_MS", "3,8,11,15,16,17,20,21,24,32").split(",")]
for M in Ms:
    bosrm.bos_rootmusic_demod(st, M, flags=True)
    bosrm.bos_rootmusic_demod_ex(st, M, flags=True)
    print("M", M, flush=True)
for M in (8, 19, 24):
    bosrm.bos_rootmusic_demod_variant(st[:2], M, variant=bosrm.VARIANT_FB, flags=True, omega=True)
for M, m in ((8, 3), (12, 5)):
    bosrm.bos_rootmusic_demod_variant(st[:2], M, variant=bosrm.VARIANT_PAPER, flags=True, omega=True,
                                      subarray_len=m)
bosrm.bos_rootmusic_demod_variant(st[:1, :20, :40].contiguous(), 8, variant=bosrm.VARIANT_FP64, flags=True)
print("variants", flush=True)
bosrm.bos_rootmusic_demod_stack(st, 8, ref_index=1, flags=True)
bosrm.bos_rootmusic_iteration_counts(st, 8)
h = st.cpu().pin_memory()
bosrm.bos_rootmusic_demod_stack_host(h, 8, ref_index=0, h_flags=True, chunk_frames=2)
u8 = torch.stack([synth.make_intensity_frame(w, t, device=dev) for t in range(3)])
g = bosrm.bos_analytic_signal(u8, synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
plan = bosrm.AnalyticPlan(w.H, w.W, 3)
g2 = bosrm.bos_analytic_signal_planned(plan, u8, synth.CARRIER_FX, synth.CARRIER_FY, 0.05, False)
torch.cuda.synchronize()
plan.close()
ph, _ = bosrm.bos_rootmusic_demod(g, 8)
bosrm.bos_unwrap(ph)
bosrm.bos_index_gradient(ph, 1.333, 1.0, 1e4, 0.01)
bosrm.bos_vertical_profile(ph)
torch.cuda.synchronize()
print("sanitize smoke done")
