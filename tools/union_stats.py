"""CPU estimate of the FSAI pair-union structure: for N uniform
points in the unit cube with the lower kNN pattern (w = 100, index order), the
spatial cell-tile order of fsai_sddmm.cu (or Morton), groups of GA consecutive
points -> needed S pairs per row (pairs kept by the spatially later point),
evaluated D entries per row, and the fraction of 8x8 DMMA tiles of the
position-sorted union that hold a needed pair.
    python tools/union_stats.py N GA [raster|morton]
(N = 20000, GA = 32: 367 needed / 1221 evaluated per row, 0.30; 86 % of the
tiles are touched -- tile skipping would save little)"""
import numpy as np, sys
from scipy.spatial import cKDTree
rng=np.random.default_rng(0)
N=int(sys.argv[1]); w=100; GA=int(sys.argv[2]) if len(sys.argv)>2 else 32
X=rng.random((N,3))
# lower kNN pattern: J_i = i + (w-1) nearest among j<i
J=[]
tree_all=cKDTree(X)
for i in range(N):
    if i < w:
        J.append(np.arange(i+1)); continue
    kq=min(i, 4*w)
    while True:
        d,idx=tree_all.query(X[i], k=min(N,kq*int(N/i)+w) if i<N else kq)
        idx=idx[idx<i]
        if len(idx)>=w-1: break
        kq*=2
    J.append(np.sort(np.append(idx[:w-1],i)))
# spatial order: cells ~2 points, 4x4x4 tiles
gper=int(np.ceil((N/2)**(1/3))); t=min(4,gper); g=((gper+t-1)//t)*t; nb=g//t
cc=np.minimum((X*g).astype(int),g-1)
b=cc//t; l=cc%t
key=((b[:,2]*nb+b[:,1])*nb+b[:,0])*(t**3)+(l[:,2]*t+l[:,1])*t+l[:,0]
ORDER=sys.argv[3] if len(sys.argv)>3 else 'raster'
if ORDER=='morton':
    def spread(v):
        r=np.zeros_like(v)
        for bit in range(11):
            r|=((v>>bit)&1)<<(3*bit)
        return r
    key=spread(cc[:,0])|(spread(cc[:,1])<<1)|(spread(cc[:,2])<<2)
sorder=np.argsort(key,kind='stable'); pos=np.empty(N,int); pos[sorder]=np.arange(N)
# B_a
B=[set() for _ in range(N)]
for i in range(N):
    Ji=J[i]
    for a in Ji:
        pa=pos[a]
        B[a].update(int(x) for x in Ji if pos[x]<=pa)
need=sum(len(s) for s in B)
G=(N+GA-1)//GA
totD=0; tiles=0; tiles_needed=0
for gi in range(G):
    rows=sorder[gi*GA:(gi+1)*GA]
    U=set()
    for a in rows: U|=B[a]
    U=np.array(sorted(U,key=lambda x:pos[x]))
    totD+=len(rows)*len(U)
    col={int(u):c for c,u in enumerate(U)}
    M=np.zeros((len(rows),len(U)),bool)
    for r,a in enumerate(rows):
        for bb in B[a]: M[r,col[bb]]=True
    for r0 in range(0,len(rows),8):
        for c0 in range(0,len(U),8):
            tiles+=1; tiles_needed+=M[r0:r0+8,c0:c0+8].any()
print(f"{ORDER} N={N} GA={GA} needed pairs {need} ({need/N:.0f}/row)  D entries {totD} ({totD/N:.0f}/row)  eff {need/totD:.2f}  tiles needed {tiles_needed}/{tiles} = {tiles_needed/tiles:.2f}")
