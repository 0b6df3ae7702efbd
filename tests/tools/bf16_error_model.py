"""Error model: the discriminator step with bf16-rounded GEMM operands and exact
accumulation vs the fp64 oracle (derives the BF16 tolerances in DESIGN.md)."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))
from oracle import gan, mlp, proxy
def bf16(x):
    x=np.asarray(x,np.float32); u=x.view(np.uint32).astype(np.uint64)
    r=((u+0x7FFF+((u>>16)&1))>>16)<<16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
Q=None
def mm(a,b,hidden):
    if not hidden or Q is None: return a@b
    return bf16(a)@bf16(b)
def fwd(Ws,bs,x):
    h=x; cache=[]; L=len(Ws)
    for l in range(L):
        z=mm(h,Ws[l].T, 0<l<L-1)+bs[l]; cache.append((h,z)); h=mlp.lrelu(z) if l<L-1 else z
    return h,cache
def bwd(Ws,cache,dout):
    L=len(Ws); g=dout; dW=[None]*L
    for l in reversed(range(L)):
        h,z=cache[l]; d=g if l==L-1 else g*mlp.lrelu_grad(z)
        dW[l]=mm(d.T,h,0<l<L-1); g=mm(d,Ws[l],0<l<L-1)
    return dW,g
def step(q):
    global Q; Q=q
    cfg=gan.paper_config(param_samples=64,events_per_sample=64,reference_rows=8192,shard_rows=4096,seed=4)
    st=gan.RankState(cfg,0); out=gan.local_step(cfg,gan.RankState(cfg,0),0)
    N=cfg.n_events; X=np.concatenate([out['x'],out['y']]); t=np.r_[np.ones(N),np.zeros(N)]
    z,c=fwd(st.dW,st.db,X); z=z[:,0]; ld=mlp.bce_with_logits(z,t)
    dW,_=bwd(st.dW,c,mlp.bce_grad(z,t)[:,None])
    W2=[w.copy() for w in out['dW_d']]  # not used
    # G step with D after adam from oracle (use oracle's updated D from a fresh run)
    st2=gan.RankState(cfg,0); o2=gan.local_step(cfg,st2,0)
    z,c=fwd(st2.dW,st2.db,out['y']); z=z[:,0]; lg=mlp.bce_with_logits(z,np.ones(N))
    _,dy=bwd(st2.dW,c,mlp.bce_grad(z,np.ones(N))[:,None])
    return ld,lg,np.concatenate([w.ravel() for w in dW]),dy
r=step(None); b=step('bf16')
rel=lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
print("loss_d",abs(b[0]-r[0])/r[0],"loss_g",abs(b[1]-r[1])/r[1],"dW_D",rel(b[2],r[2]),"dy",rel(b[3],r[3]))
