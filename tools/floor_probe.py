"""Why the C2 oracle self-floor is 1.2e-9 (SURVEY's numpy probe: ~5e-11): the same 1-vs-8-row-shard
Gram experiment with the oracle's sequential per-element sums and with BLAS's blocked sums (CPU only)."""
import sys, numpy as np, time
sys.path.insert(0,'.')
import oracle, paper_2011_02436_b200 as rb
oracle.set_threads(8)
n,d,L,m=50000,64,1000,10
x,t=rb.synth_classification(n,d,m,1001,2001)
w,b=oracle.init_hidden(d,L,m,3001)
h=oracle.hidden_matrix(w,b,x)
def solve_from(g, hty):
    order,rank,_,f,_=oracle.factor_gram(g, n)
    xs=oracle.solve_factored_gram(f,order,rank,hty[order]); beta=np.empty_like(xs); beta[order]=xs; return beta
rel=lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
# oracle sequential sums
g1=oracle.gram(h,1); g8=oracle.gram(h,8)
hty1=h.T@t  # same for both (isolate the Gram)
b1=solve_from(g1,hty1); b8=solve_from(g8,hty1)
print("oracle sequential Gram, 1 vs 8 shards: beta rel", rel(b8,b1), " G rel", rel(g8,g1))
# BLAS (blocked, FMA) Gram
G1=h.T@h; G8=sum(h[i*6250:(i+1)*6250].T@h[i*6250:(i+1)*6250] for i in range(8))
G1=np.tril(G1)+np.tril(G1,-1).T; G8=np.tril(G8)+np.tril(G8,-1).T
B1=solve_from(G1,hty1); B8=solve_from(G8,hty1)
print("BLAS Gram, 1 vs 8 shards: beta rel", rel(B8,B1), " G rel", rel(G8,G1))
print("oracle vs BLAS 1-shard: beta rel", rel(B1,b1), " G rel", rel(G1,g1))
print("cond(H) ~", np.sqrt(np.linalg.cond(G1)))
