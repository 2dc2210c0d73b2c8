"""C2 backward footprint at 4-B, 32-B, 64-B and 128-B granularity (first 6 examples,
untransformed): the DRAM-read floor of an atom-centric backward over the (N,C,D,D,D)
layout.  Round 2: 40.8 / 56.5 / 67.2 / 79.6 MB per 50-grid step vs 83 MB measured."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, bench
cfg=bench.CONFIGS['c2']; exs,_=bench.make_batch(cfg,0,1)
D=48; res=0.5; rmult=1.5
tot_vox=0; tot_sec=0; T64=[]; T128=[]
for ex in exs[:6]:
    sets=ex.coord_sets
    center=sets[-1].coords.astype(np.float64).mean(axis=0); origin=center-11.75
    choff=0; vox=set(); sec=set(); s64=set(); s128=set()
    for cs in sets:
        xyz=cs.coords.astype(np.float64)-origin; r=cs.radii.astype(np.float64)*rmult
        for a in range(len(xyz)):
            x,y,z=xyz[a]; c=r[a]; ch=choff+int(cs.type_index[a])
            lo=np.ceil((xyz[a]-c)/res).clip(0,None).astype(int); hi=np.floor((xyz[a]+c)/res).clip(None,D-1).astype(int)
            if (lo>hi).any(): continue
            I=np.arange(lo[0],hi[0]+1); J=np.arange(lo[1],hi[1]+1); K=np.arange(lo[2],hi[2]+1)
            dx=I*res-x; dy=J*res-y; dz=K*res-z
            d2=dx[:,None,None]**2+dy[None,:,None]**2+dz[None,None,:]**2
            ii,jj,kk=np.nonzero(d2<c*c)
            addr=((ch*D+I[ii])*D+J[jj])*D+K[kk]
            vox.update(addr.tolist()); sec.update((addr//8).tolist()); s64.update((addr//16).tolist()); s128.update((addr//32).tolist())
        choff+=cs.num_types
    tot_vox+=len(vox); tot_sec+=len(sec); T64.append(len(s64)); T128.append(len(s128))
n=6
print("footprint per grid: voxels", tot_vox/n, "bytes", 4*tot_vox/n, "sector bytes", 32*tot_sec/n, "ratio", 32*tot_sec/(4*tot_vox))
print("per 50-grid step: 4F MB", 4*tot_vox/n*50/1e6, "sector MB", 32*tot_sec/n*50/1e6)
print("64B MB", 64*sum(T64)/n*50/1e6, "128B MB", 128*sum(T128)/n*50/1e6)
