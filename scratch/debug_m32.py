import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth
M = 32
w = synth.workload("C4", H=2048, W=2048)
frames = synth.make_stack(w, frames=range(8), device="cuda")
raw, fl = bosrm.bos_rootmusic_demod(frames, M, flags=True)
torch.cuda.synchronize()
rng = np.random.default_rng(M)
pix = (rng.integers(0, 2048, 4096), rng.integers(0, 2048, 4096))
host = frames[[0, 7]].cpu().numpy()
for j, t in enumerate([0, 7]):
    win, _ = R.extract_windows(host[j], pix[0], pix[1], M)
    res = R.estimate_windows(win)
    g = raw[t].cpu().numpy()[pix]
    gf = fl[t].cpu().numpy()[pix]
    e = np.abs(R.wrap(g - res["alpha"]))
    ok = (res["flags"] & 0x1f) == 0
    bad = np.argsort(np.where(ok, e, 0))[::-1][:32]
    print(f"frame {t}: n bad >1e-2:", ((e > 1e-2) & ok).sum(), "of", e.size, "oracle-flagged", (~ok).sum(), "gpu flagged", (gf & 0x1f != 0).sum())
    print("  errs", np.round(e[bad][:8], 4), "gflags", gf[bad][:8], "margin", np.round(res["margin"][bad][:8], 4))
    np.savez(f"gpurun_out/m32_bad_f{t}.npz", win=win[bad], gpu=g[bad], ora=res["alpha"][bad], px=pix[1][bad], py=pix[0][bad], err=e[bad])
