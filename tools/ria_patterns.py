"""Count the runs and distinct run patterns (18 relative offsets of the
scatter adjacency, list_lattice.cpp:206-226) of a cubic blocks lattice with
numpy -- sizes the pattern-id coding of the RIA odd step.

    python tools/ria_patterns.py NX BLOCK SPACING     # e.g. 400 8 8 (cfg 4)
"""
import numpy as np, sys
nx=ny=nz=int(sys.argv[1]); b=int(sys.argv[2]); s=int(sys.argv[3])
x=np.arange(nx)%(b+s)>=s; y=np.arange(ny)%(b+s)>=s; z=np.arange(nz)%(b+s)>=s
solid=x[:,None,None]&y[None,:,None]&z[None,None,:]
fluid=~solid
rank=np.cumsum(fluid.ravel(),dtype=np.int64).reshape(nx,ny,nz)-1
rank=rank.astype(np.int64)
N=int(fluid.sum())
own=rank[fluid]
C=[(1,0,0),(-1,0,0),(0,1,0),(0,-1,0),(0,0,1),(0,0,-1),(1,1,0),(-1,-1,0),(1,-1,0),(-1,1,0),(1,0,1),(-1,0,-1),(1,0,-1),(-1,0,1),(0,1,1),(0,-1,-1),(0,1,-1),(0,-1,1)]
cols=[]
for d,(cx,cy,cz) in enumerate(C):
    nb_f=np.roll(fluid,(-cx,-cy,-cz),axis=(0,1,2))
    nb_r=np.roll(rank,(-cx,-cy,-cz),axis=(0,1,2))
    v=np.where(nb_f, nb_r-rank, -(1<<40)-d)[fluid]
    cols.append(v)
P=np.stack(cols,1)
u=np.unique(P,axis=0)
chg=np.any(P[1:]!=P[:-1],axis=1)
print("N",N,"runs",int(chg.sum())+1,"distinct",len(u))
