"""Config 3 design study (CPU only): lockstep steps of the irregular kernel's
K-groups against an in-band linked-list walk (leaf records pointing at the
next tree's root, lanes free-running inside a window of ring stages).
Path lengths come from config 3's own trees and rows (synth.config3).
Output: profiles/r2_cstream_list_walk_simulation.txt.

    python tools/sim_cstream_steps.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_2287_b200 import synth
T=640
w = synth.config3(n=1, trees=T); fl = w.flat
depths = fl.depths()
n = 256
X = synth.hash_uniform(w.hash_seed, 0, n, 700, 0.4)
PL = np.zeros((T, n), np.int32)
for t in range(T):
    a, b = int(fl.tree_off[t]), int(fl.tree_off[t+1])
    fid, val, lc, rc = fl.fid[a:b], fl.value[a:b], fl.left[a:b], fl.right[a:b]
    cur = np.zeros(n, np.int64); L = np.zeros(n, np.int32)
    while True:
        f = fid[cur]; live = f >= 0
        if not live.any(): break
        x = X[np.arange(n), np.where(live, f, 0)]
        nxt = np.where(x >= val[cur], rc[cur], lc[cur])
        cur = np.where(live, nxt, cur); L += live
    PL[t] = L
np.save('/tmp/PL.npy', PL); np.save('/tmp/depths.npy', depths)

# ---- step counts
PL = np.load('/tmp/PL.npy'); depths = np.load('/tmp/depths.npy')
T, n = PL.shape
def lockstep(K, C=64):
    tot = 0
    for c0 in range(0, T, C):
        idx = np.arange(c0, min(T, c0+C))
        order = idx[np.argsort(depths[idx], kind='stable')]
        for g in range(0, len(order), K):
            tot += depths[order[g:g+K]].max() * K
    return tot * (n//32)   # chain-level issue units, per 32-row tile summed
def lists(S, K, C, nst, extra=1):
    # S warps, K chains -> L lists; chunk of C trees; window nst chunks
    L = S*K
    total = 0
    nch = T // C
    for tile in range(n//32):
        pl = PL[:, tile*32:(tile+1)*32] + extra   # steps per tree incl leaf step
        # list l has trees: for chunk c: slots j with j % L == l -> tree c*C + j
        per = [[ [c*C + j for j in range(l, C, L)] for c in range(nch)] for l in range(L)]
        # state per (list, lane): chunk idx, pos in chunk list, remaining steps
        ch = np.zeros((L,32), np.int64); pos = np.zeros((L,32), np.int64)
        rem = np.zeros((L,32), np.int64)
        def load(l, r):
            while ch[l,r] < nch and pos[l,r] >= len(per[l][ch[l,r]]):
                ch[l,r] += 1; pos[l,r] = 0
            if ch[l,r] < nch:
                rem[l,r] = pl[per[l][ch[l,r]][pos[l,r]], r]
        for l in range(L):
            for r in range(32): load(l, r)
        oldest = 0; steps = 0
        while True:
            if (ch >= nch).all(): break
            oldest = ch.min()
            active = (ch < nch) & (ch < oldest + nst)
            # per warp: any active lane-chain -> warp issues K chain-steps
            wa = active.reshape(S, K, 32).any(axis=(1,2))
            steps += wa.sum() * K
            rem[active] -= 1
            done = active & (rem == 0)
            for l, r in zip(*np.nonzero(done)):
                pos[l,r] += 1; load(l, r)
        total += steps
    return total
base = lockstep(3)
print("lockstep K=3 C=64:", base, " K=2:", lockstep(2), "K=4", lockstep(4))
true = (PL.sum()/32)
print("true visits (warp units)", true, "eff of lockstep", true/base)
for (S,K,C,nst) in [(16,3,64,2),(16,2,64,2),(16,2,32,4),(16,1,64,2),(16,1,32,4),(16,1,16,8),(8,2,16,8),(16,3,48,2),(16,2,32,3)]:
    r = lists(S,K,C,nst)
    print((S,K,C,nst), r, "vs lockstep", base/r)
