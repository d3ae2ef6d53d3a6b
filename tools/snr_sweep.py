"""Throughput and iteration counts of the M=8 demod vs SNR on C3 frames (plus the f1 front-end output)."""
import torch, sys, json
sys.path.insert(0, '.')
from paper_1910_11872_b200 import bosrm, synth
dev = "cuda"
w = synth.workload("C3")
def timeit(fr, M=8):
    out = torch.empty(fr.shape, dtype=torch.float32, device=dev)
    bosrm.bos_rootmusic_demod(fr, M, out_phase=out); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): bosrm.bos_rootmusic_demod(fr, M, out_phase=out)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    c = bosrm.bos_rootmusic_iteration_counts(fr, M)
    n = c["pixels"]
    return dict(mpix_s=round(fr.numel() / ms / 1e3, 1), power=round(c["power_its"] / n, 2), aby=round(c["aberth_y"] / n, 3), abx=round(c["aberth_x"] / n, 3))
for snr in (0.0, 10.0, 20.0, 30.0, 40.0, None):
    fr = synth.make_stack(w, frames=[5, 50], device=dev, snr_db=snr)
    print("snr", snr, timeit(fr))
u8 = torch.stack([synth.make_intensity_frame(w, t, device=dev) for t in (5, 50)])
g = bosrm.bos_analytic_signal(u8, synth.CARRIER_FX, synth.CARRIER_FY, 0.05)
print("f1 output", timeit(g))
