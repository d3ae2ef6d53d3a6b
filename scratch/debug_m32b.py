import numpy as np, torch, sys, math
sys.path.insert(0, '.')
from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth
M = 32; T = 8
w = synth.workload("C4", H=2048, W=2048)
frames = synth.make_stack(w, frames=range(T), device="cuda")
ref, _ = bosrm.bos_rootmusic_demod(frames[0:1], M); ref = ref[0].contiguous()
out = torch.empty(T, 2048, 2048, dtype=torch.float32, device="cuda")
bosrm.bos_rootmusic_demod(frames, M, ref_phase=ref, out_phase=out)
raw, _ = bosrm.bos_rootmusic_demod(frames, M)
torch.cuda.synchronize()
d = (out - torch.remainder(raw - ref + math.pi, 2 * math.pi) + math.pi)
d = torch.remainder(out - (raw - ref) + math.pi, 2*math.pi) - math.pi
print("max |out - wrap(raw-ref)| per frame:", [float(d[t].abs().max()) for t in range(T)])
bad = (d.abs() > 1e-3).nonzero()
print("n bad:", bad.shape[0], bad[:10].tolist())
# raw vs oracle on the bad pixels of frame 7
if bad.shape[0]:
    b = bad[bad[:,0]==7][:16].cpu().numpy()
    py, px = b[:,1], b[:,2]
    host = frames[[0,7]].cpu().numpy()
    o, ofl = R.demod_stack(host, M, pixels=(py,px), frame_indices=[1])
    print("oracle vs out:", np.round(R.wrap(out[7].cpu().numpy()[py,px]-o[0]),4))
    print("oracle vs raw-ref:", np.round(R.wrap((raw[7]-ref).cpu().numpy()[py,px]-o[0]),4))
