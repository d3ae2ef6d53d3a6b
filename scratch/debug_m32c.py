import numpy as np, torch, sys, math, time
sys.path.insert(0, '.')
from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth
M = 32; T = 8
w = synth.workload("C4", H=2048, W=2048)
frames = synth.make_stack(w, frames=[0, 7], device="cuda")
raw, fl = bosrm.bos_rootmusic_demod(frames, M, flags=True)
torch.cuda.synchronize()
rng = np.random.default_rng(M)
pix = (rng.integers(0, 2048, 1024), rng.integers(0, 2048, 1024))
host = frames.cpu().numpy()
for t in (0, 1):
    win, _ = R.extract_windows(host[t], pix[0], pix[1], M)
    res = R.estimate_windows(win)
    g = raw[t].cpu().numpy()[pix]
    e = np.abs(R.wrap(g - res["alpha"]))
    ok = (res["flags"] & 0x1f) == 0
    bad = np.nonzero((e > 1e-3) & ok)[0]
    print(f"t={t}: bad {bad.size}: err {np.round(e[bad],4)} margin {np.round(res['margin'][bad],4)} gfl {fl[t].cpu().numpy()[pix][bad]} px {pix[1][bad]} py {pix[0][bad]}")
    np.savez(f"gpurun_out/m32c_t{t}.npz", win=win[bad], gpu=g[bad], ora=res["alpha"][bad], margin=res["margin"][bad])
