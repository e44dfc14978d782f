"""Bank-conflict model of the C3 stride-table gathers: wavefronts per warp
lookup (max distinct 4-byte words per bank over 32 lanes) for C3's own
state/word distribution at K = 2 step boundaries, under the device layout
(column-major, accepting states first), an XOR row swizzle, frequency
renumbering, and uniformly random addresses.  CPU only:
    python tools/bank_sim.py
Result (4 Mi bases): device 3.55, swizzle 3.51, by-frequency 3.53, uniform 3.53
(ncu measured 3.56 on the B200)."""
import sys

import numpy as np

sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
from paper_1509_01506_b200 import workloads
import paper_1509_01506_b200 as ks
w = workloads.make(3, 1<<22)
d = w.dfa; T = d.transitions
codes = ks.encode_bytes(w.ascii.tobytes())
# states at even positions (K=2 steps), skip N regions
n = codes.size
s = 0; S=[]; W=[]
states = np.empty(n, np.int32)
for i in range(n):
    s = T[s, codes[i]]; states[i]=s
# step j: from state at pos 2j-1 with word (c[2j], c[2j+1])
prev = states[1:-2:2]; c0 = codes[2::2][:prev.size]; c1 = codes[3::2][:prev.size]
ok = (c0<4)&(c1<4)
prev=prev[ok]; wd=(c0[ok] | (c1[ok]<<2)).astype(np.int64)
acc = np.diff(d.out_offsets)>0
Q = d.state_count
# device numbering: accepting first (stable order) then the rest
order = np.concatenate([np.nonzero(acc)[0], np.nonzero(~acc)[0]])
newid = np.empty(Q, np.int64); newid[order]=np.arange(Q)
freq = np.bincount(prev, minlength=Q)
byfreq = np.argsort(-freq, kind='stable'); fid = np.empty(Q,np.int64); fid[byfreq]=np.arange(Q)
rng = np.random.default_rng(0)
def sim(ids, swz):
    tot=0; trials=20000
    for t in range(trials):
        idx = rng.integers(0, prev.size, 32)
        sid = ids[prev[idx]]; ww = wd[idx]
        row = sid ^ (ww<<1) if swz==1 else sid ^ ww if swz==2 else sid
        word = (ww<<11) | (row>>1)     # 4-byte word index
        bank = word & 31
        # wavefronts = max over banks of distinct words
        m=0
        for b in np.unique(bank):
            m=max(m, np.unique(word[bank==b]).size)
        tot+=m
    return tot/trials
for name, ids in (("orig",np.arange(Q)),("device(acc-first)",newid),("by-freq",fid)):
    for swz in (0,1):
        print(name, "swizzle" if swz else "plain", round(sim(ids,swz),3))
# uniform random baseline
tot=0
for t in range(20000):
    word = rng.integers(0, 1<<15, 32); bank = word & 31
    tot += max(np.unique(word[bank==b]).size for b in np.unique(bank))
print("uniform", tot/20000)
