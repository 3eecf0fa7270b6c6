"""Config 3 design study (CPU only): shared-memory wavefronts per warp-tree of
the irregular kernel's lockstep K-groups against the in-band linked-list walk
(tools/sim_cstream_steps.py), from the records' real addresses: an LDS.64 of
32 lanes is served in two half-warp phases, each costing the largest number
of distinct 8-byte words that fall into one bank pair.
Output: profiles/r2_cstream_list_walk_simulation.txt.

    python tools/sim_cstream_wavefronts.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_2287_b200 import synth
T=256; C=64
w = synth.config3(n=1, trees=T); fl = w.flat
depths = fl.depths()
n = 128
X = synth.hash_uniform(w.hash_seed, 0, n, 700, 0.4)
# BFS layout per tree (sibling pairs adjacent), record index within tree
trees=[]
for t in range(T):
    a, b = int(fl.tree_off[t]), int(fl.tree_off[t+1])
    fid, val, lc, rc = fl.fid[a:b], fl.value[a:b], fl.left[a:b], fl.right[a:b]
    order=[0]; newid={0:0}
    h=0
    while h < len(order):
        i=order[h]; h+=1
        if fid[i] < 0: continue
        newid[lc[i]]=len(order); order.append(lc[i]); newid[rc[i]]=len(order); order.append(rc[i])
    nf = np.array([fid[i] for i in order]); nv=np.array([val[i] for i in order])
    nl = np.array([newid[lc[i]] if fid[i]>=0 else k for k,i in enumerate(order)])
    trees.append((nf,nv,nl,len(order)))
# paths: for each tree, each row: list of record indices visited (internal nodes), then leaf index
def path(t, r):
    nf,nv,nl,_=trees[t]
    k=0; p=[]
    while nf[k]>=0:
        p.append(k); k = nl[k] + (1 if X[r,nf[k]]>=nv[k] else 0)
    return p, k
paths = [[path(t,r) for r in range(n)] for t in range(T)]
def wf64(addrs):
    # addrs: list of 8-byte record indices (global in stage) for active lanes (lane order matters: half-warps)
    tot=0
    for half in (addrs[:16], addrs[16:]):
        half=[x for x in half if x is not None]
        if not half: continue
        d={}
        for x in set(half): d.setdefault(x%16,[]).append(x)
        tot+=max(len(v) for v in d.values())
    return tot
# stage record base per tree in chunk
def chunk_base(c0):
    base={}; o=0
    for t in range(c0, c0+C):
        base[t]=o; o+= (trees[t][3]+1)//2*2
    return base
def lockstep(K):
    steps=0; wf=0
    for c0 in range(0,T,C):
        base=chunk_base(c0)
        idx=list(range(c0,c0+C)); idx.sort(key=lambda t:-depths[t])
        for g in range(0,C,K):
            ts=idx[g:g+K]; dmax=max(depths[t] for t in ts)
            for tile in range(n//32):
                for t in ts:
                    for l in range(dmax):
                        steps+=1
                        ad=[]
                        for r in range(tile*32,tile*32+32):
                            p,leaf=paths[t][r]
                            if l < len(p): ad.append(base[t]+p[l])
                            elif l==len(p): ad.append(base[t]+leaf)   # loads leaf record once (live), then parked
                            else: ad.append(None)
                        w_=wf64(ad)
                        wf+= w_ + (1 if w_ else 0)
                    wf+=2  # leaf value read + store
    return steps, wf
def lists(S,K):
    L=S*K; steps=0; wf=0
    for c0 in range(0,T,C):
        base=chunk_base(c0)
        idx=list(range(c0,c0+C)); idx.sort(key=lambda t:-depths[t])
        per=[idx[l::L] for l in range(L)]
        for tile in range(n//32):
            for s in range(S):
                # warp s: chains k -> list s*K+k; per lane sequence of addresses
                seqs=[]
                for k in range(K):
                    sq=[]
                    for r in range(tile*32,tile*32+32):
                        a=[]
                        for t in per[s*K+k]:
                            p,leaf=paths[t][r]
                            a += [(base[t]+x,0) for x in p] + [(base[t]+leaf,1)]
                        sq.append(a)
                    seqs.append(sq)
                nst=max(len(a) for sq in seqs for a in sq)
                for i in range(nst):
                    for k in range(K):
                        steps+=1
                        ad=[sq[i][0] if i<len(sq) else -1 for sq in seqs[k]]  # parked lanes read park record (same addr)
                        anyleaf=any(i<len(sq) and sq[i][1] for sq in seqs[k])
                        wf+= wf64(ad) + 1 + (1 if anyleaf else 1)  # park stores too
    return steps, wf
ntr = T*(n//32)
for K in (2,3):
    s,wv=lockstep(K); print("lockstep K",K,"steps/warp-tree",s/ntr,"wf/warp-tree",wv/ntr)
for S,K in ((16,1),(16,2),(16,3)):
    s,wv=lists(S,K); print("lists",S,K,"steps/warp-tree",s/ntr,"wf/warp-tree",wv/ntr)
