"""Distinct 128-byte lines per warp LDG.256 of the binned C3 quad eval: bins in
random order vs sorted by cell (eval).  CPU only."""
import numpy as np
rng=np.random.default_rng(0)
S=253; nb=32; n=1<<24
N=2000*512  # simulate ~2000 bins worth: restrict points to first bins region to save time
u,v,w=(rng.random(n).astype(np.float32) for _ in range(3))
bu=np.minimum((u*nb).astype(int),nb-1); bv=np.minimum((v*nb).astype(int),nb-1); bw=np.minimum((w*nb).astype(int),nb-1)
b=(bw*nb+bv)*nb+bu
sel=b<2000
u,v,w,b,bu,bv,bw=u[sel],v[sel],w[sel],b[sel],bu[sel],bv[sel],bw[sel]
c=[np.clip(((q*nb-bq)*8).astype(int),0,7) for q,bq in ((u,bu),(v,bv),(w,bw))]
key=(c[2]*8+c[1])*8+c[0]
order=np.lexsort((key,b))
su=np.minimum((u*S).astype(int),S-1)[order]; sv=np.minimum((v*S).astype(int),S-1)[order]; sw=np.minimum((w*S).astype(int),S-1)[order]
bo=b[order]
EU,EV,EW=16,19,19
def entry(su,sv,sw):
    bx,by,bz=su>>4,sv>>4,sw>>4
    lu,lv,lw=su&15,sv&15,sw&15
    brick=(bz*16+by)*16+bx
    return (brick*EU*EV*EW+(lw*EV+lv)*EU+lu)*32
# warps: per bin, 128-thread CTA, warps of 32 consecutive sorted points
starts=np.r_[0,np.flatnonzero(np.diff(bo))+1,len(bo)]
def wavefronts(L, G):   # distinct lines per aligned group of G lanes, summed
    return sum(len(np.unique(L[g:g + G])) for g in range(0, len(L), G))
tot = {32: [0, 0], 4: [0, 0]}; ninst = 0
for i in range(len(starts) - 1):
    a, z = starts[i], starts[i + 1]
    idx = np.arange(a, z)
    rnd = rng.permutation(idx)
    for wb in range(a, z, 32):
        for k, ids in enumerate((idx[wb - a:wb - a + 32], rnd[wb - a:wb - a + 32])):
            for bb in (0, 2):
                for cc in range(4):
                    L = entry(su[ids], sv[ids] + bb, sw[ids] + cc) // 128
                    for G in (32, 4):
                        tot[G][k] += wavefronts(L, G)
                    ninst += k == 0
for G in (32, 4):
    print(f"lane groups of {G}: sorted {tot[G][0] / ninst:.1f}, random bin order {tot[G][1] / ninst:.1f} lines per LDG.256")
