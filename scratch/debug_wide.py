import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth
for M in (19, 32, 24):
    H, W = M + 6, 75
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=M), 5, snr_db=10.0)
    g, fl = bosrm.bos_rootmusic_demod(f.to("cuda"), M, flags=True)
    torch.cuda.synchronize()
    g = g.cpu().numpy()[0]; fl = fl.cpu().numpy()[0]
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    win, _ = R.extract_windows(f.numpy(), yy.ravel(), xx.ravel(), M)
    res = R.estimate_windows(win)
    o = res["alpha"].reshape(H, W); ofl = res["flags"].reshape(H, W)
    e = np.abs(R.wrap(g - o)); ok = (ofl & 0x1f) == 0
    e[~ok] = 0
    idx = np.argsort(e.ravel())[::-1][:8]
    print(f"M={M} rms={np.sqrt(np.mean(e[ok]**2)):.2e} max={e.max():.2e}")
    # error vs position within 32-px segment
    seg = xx % 32
    for s0 in (0, 1, 2, 8, 16, 31):
        m = ok & (seg == s0)
        if m.any(): print(f"   seg pos {s0}: rms {np.sqrt(np.mean(e[m]**2)):.2e} max {e[m].max():.2e}")
    for i in idx:
        y, x = divmod(i, W)
        print(f"   px ({y},{x}) err {e[y,x]:.3e} gflag {fl[y,x]} margin {res['margin'][i]:.3e} gap {(res['S'][i,0]/res['S'][i,1])**2:.2f} |c|/norm {abs(res['c'][i]):.3f}")
