exec(open('/tmp/emu_wide.py').read().split("M=32; H,W")[0])
import numpy as np
dat=np.load('/root/repo/gpurun_out/m32c_t1.npz')
win=dat['win']; M=32
print("gpu", dat['gpu'], "oracle", dat['ora'], "margin", dat['margin'])
ref=R.estimate_windows(win)
w32=win.astype(c64); Rm=w32@np.conj(np.swapaxes(w32,1,2))
_,V=np.linalg.eigh(Rm.astype(np.complex128)); u=V[:,:,-1].astype(c64)
v=np.einsum("nik,ni->nk",np.conj(w32),u); v=(v/np.linalg.norm(v,axis=1,keepdims=True)).astype(c64)
T=E.template(M).astype(c64)[:M-1]
# oracle roots
U,S,Vh=R.svd_subspaces(win); Cy,Cx=R.noise_projectors(U,Vh)
for name,q,C in (("y",u,Cy),("x",v,Cx)):
    c,rot=E.coeffs(q)
    z,it=aberth_jacobi(c,T[None,:]*rot[:,None],tol2=1e-3)
    ro,_=R.companion_roots(R.music_polynomial(C))
    ro=ro[0]; ro_in=ro[np.abs(ro)<=1+1e-9]
    d_or=np.sort(np.abs(np.log(np.abs(ro_in))))[:4]
    dz=np.abs(np.log(np.abs(z[0])))
    i=np.argsort(dz)[:4]
    print(name,"its",it,"oracle best d",np.round(d_or,4))
    print("   gpu-emu best d",np.round(dz[i],4),"args",np.round(np.angle(z[0][i]),3))
    j=np.argsort(np.abs(np.log(np.abs(ro_in))))[:4]
    print("   oracle args",np.round(np.angle(ro_in[j]),3))
print("---- tight")
for name,q,C in (("y",u,Cy),):
    c,rot=E.coeffs(q)
    for tol in (1e-3,1e-6,1e-10):
        z,it=aberth_jacobi(c,T[None,:]*rot[:,None],tol2=tol)
        dz=np.abs(np.log(np.abs(z[0]))); i=np.argsort(dz)[:3]
        zb=z[0][i[0]]
        zp=zb
        for k in range(6):
            w=E.newton_ratio(c,np.array([zp]).astype(c64))[0]; zp=zp-w
        print(tol,"its",it,"best d",np.round(dz[i],4),"args",np.round(np.angle(z[0][i]),3),"polished",np.round(np.abs(np.log(abs(zp))),4),np.round(np.angle(zp),3),"moved",abs(zp-zb))
