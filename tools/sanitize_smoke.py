"""Small invocation of every entry point, for compute-sanitizer (memcheck / racecheck /
initcheck / synccheck — one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1910_11872_b200 import bosrm, synth  # noqa: E402

dev = "cuda"
w = synth.workload("C3", H=37, W=70)
st = synth.make_stack(w, frames=[0, 3, 9], device=dev)
for M in (3, 8, 16, 17, 24):
    bosrm.bos_rootmusic_demod(st, M, flags=True)
    bosrm.bos_rootmusic_demod_ex(st, M, flags=True)
bosrm.bos_rootmusic_demod_stack(st, 8, ref_index=1, flags=True)
bosrm.bos_rootmusic_iteration_counts(st, 8)
h = st.cpu().pin_memory()
bosrm.bos_rootmusic_demod_stack_host(h, 8, ref_index=0, h_flags=True, chunk_frames=2)
u8 = torch.stack([synth.make_intensity_frame(w, t, device=dev) for t in range(3)])
g = bosrm.bos_analytic_signal(u8, synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
ph, _ = bosrm.bos_rootmusic_demod(g, 8)
bosrm.bos_unwrap(ph)
bosrm.bos_index_gradient(ph, 1.333, 1.0, 1e4, 0.01)
torch.cuda.synchronize()
print("sanitize smoke done")
