"""Shard-local DM input model (CPU, from the oracle index): per rank of an N-way block partition, the
canonical pair blocks its blocks touch and their mirrors, as contiguous runs, and the bytes moved when
gaps up to 0/8/64/512 KB are bridged. python tools/shard_io_model.py super448_200Ry 4
"""
import sys, time, collections
import numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from paper_1402_4247_b200.system import Fe3O4
from paper_1402_4247_b200.shard import partition
cfg=sys.argv[1]; N=int(sys.argv[2])
f=Fe3O4.config(cfg); t=time.time(); ix=Oracle(f.system).build_index(); print('index',time.time()-t)
norb=np.array([f.system.species[s].norb for s in f.system.species_of_atom])
pa,pb,pR,poff=ix['pair_a'],ix['pair_b'],ix['pair_R'].reshape(-1,3),ix['pair_off']
npair=len(pa)
key={ (int(pa[p]),int(pb[p]),tuple(int(x) for x in pR[p])):p for p in range(npair)}
bp,ca,cR,cm=ix['blk_ptr'],ix['cov_atom'],ix['cov_R'].reshape(-1,3),ix['cov_mask'].astype(np.uint64)
nb=ix['nblock']
cost=np.zeros(nb,dtype=np.int64); touched=[None]*nb
def canon(a,b,R):
    if a!=b: return a<b
    for x in R:
        if x!=0: return x>0
    return True
t=time.time()
for b in range(nb):
    c0,c1=int(bp[b]),int(bp[b+1]); s=set(); tot=0
    for i in range(c0,c1):
        for j in range(i,c1):
            both=int(cm[i])&int(cm[j])
            if not both: continue
            ai,aj=int(ca[i]),int(ca[j]); R=tuple(int(x) for x in (cR[j]-cR[i]))
            if canon(ai,aj,R): p=key[(ai,aj,R)]
            else: p=key[(aj,ai,tuple(-x for x in R))]
            s.add(p)
            nq=sum(1 for q in range(16) if (both>>(4*q))&0xF)
            tot+=((norb[ai]+7)&~7)*((norb[aj]+7)&~7)*4*nq
    cost[b]=tot; touched[b]=s
print('blocks',time.time()-t)
parts=partition(cost,N)
mir=ix['pair_mirror']; size=np.diff(poff)
for r,(b0,b1) in enumerate(parts):
    mine=set()
    for b in range(b0,b1): mine|=touched[b]
    mine=sorted(mine)
    need=sorted(set(mine)|set(int(mir[p]) for p in mine))
    def runs(ps):
        rs=[]
        for p in ps:
            o,n=int(poff[p]),int(size[p])
            if rs and rs[-1][0]+rs[-1][1]==o: rs[-1][1]+=n
            else: rs.append([o,n])
        return rs
    for name,ps in (('canon',mine),('canon+mirror',need)):
        rs=runs(ps); tot=sum(n for o,n in rs)
        out=[name, len(rs), round(tot*8/1e6,2)]
        for gapmax in (0, 1024, 8192, 65536):  # doubles
            m=[list(rs[0])]
            for o,n in rs[1:]:
                if o-(m[-1][0]+m[-1][1])<=gapmax: m[-1][1]=o+n-m[-1][0]
                else: m.append([o,n])
            out.append((gapmax*8//1024, len(m), round(sum(n for o,n in m)*8/1e6,2)))
        print('rank',r,out)
print('DM MB', ix['nnz']*8/1e6)
