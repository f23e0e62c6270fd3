"""Exhaustive search for the non-separable DMMA kernel's K order on R = 6 registers (NsSix in
csrc/mg_gamma.cu): a 9-edge pattern graph G0 on 6 registers (2 loops) and four injections
registers -> components whose images partition the 36 unordered pairs of 8 components, plus a
bank-quarter labelling Q that makes the per-lane-component LDS.64 conflict free.  R = 5 has no
solution (same search with R = 5)."""
import itertools, sys
R=6
pairs=[(a,b) for a in range(8) for b in range(a,8)]
pid={p:i for i,p in enumerate(pairs)}
FULL=(1<<36)-1
regpairs=[(i,j) for i in range(R) for j in range(i+1,R)]
def labelings():
    # Q: comp -> label 0..3, labels {0,1} used by exactly 4 comps
    for q in itertools.product(range(4),repeat=8):
        if sum(1 for x in q if x<2)==4: yield q
LAB=list(labelings())
def find_label(phis):
    groups=[set(phi[i] for phi in phis) for i in range(R)]
    for q in LAB:
        ok=True
        for gset in groups:
            ls=[q[c] for c in gset]
            if len(set(ls))<len(ls): ok=False;break
        if ok: return q
    return None
best=None
for edges in itertools.combinations(regpairs, 7):
    used=set([0,1])
    for e in edges: used|=set(e)
    if len(used)<R: continue
    G0=[(0,0),(1,1)]+list(edges)
    masks={}
    for phi in itertools.permutations(range(8),R):
        m=0
        for (i,j) in G0:
            a,b=phi[i],phi[j]
            if a>b:a,b=b,a
            m|=1<<pid[(a,b)]
        masks.setdefault(m,[]).append(phi)
    byfirst={}
    for m in masks:
        low=(m&-m).bit_length()-1
        byfirst.setdefault(low,[]).append(m)
    sols=[]
    def dfs(cov,chosen):
        if len(sols)>=20: return
        if len(chosen)==4:
            if cov==FULL: sols.append(list(chosen))
            return
        rest=FULL&~cov
        low=(rest&-rest).bit_length()-1
        for m in byfirst.get(low,[]):
            if m&cov: continue
            chosen.append(m); dfs(cov|m,chosen); chosen.pop()
    dfs(0,[])
    for ms in sols:
        # try all phi choices per mask (limited)
        for combo in itertools.islice(itertools.product(*[masks[m] for m in ms]),200):
            q=find_label(combo)
            if q:
                print("G0=",G0); print("PHI=",list(combo)); print("Q=",q)
                sys.exit(0)
print("none")
