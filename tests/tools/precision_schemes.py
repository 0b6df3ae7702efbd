"""Which tensor-core operand schemes meet the fp32 tolerances (loss 1e-5, grads
1e-3)?  numpy emulation of tf32 / bf16 / bf16x3 / fp16x3 / tf32x3 GEMMs in the
discriminator step against the fp64 oracle (precision)."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))
from oracle import gan, mlp, proxy
def bf16(x):
    x=np.asarray(x,np.float32); u=x.view(np.uint32).astype(np.uint64)
    r=((u+0x7FFF+((u>>16)&1))>>16)<<16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
def f16(x): return np.asarray(x,np.float16).astype(np.float64)
def tf32(x):
    x=np.asarray(x,np.float32); u=x.view(np.uint32).astype(np.uint64)
    r=((u+0xFFF+((u>>13)&1))>>13)<<13
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
def split(x,q,scale=1.0):
    hi=q(x); lo=q((x-hi)*scale)/scale; return hi,lo
def mm(a,b,mode):
    # a [M,K], b [K,N]
    if mode=='f64': return a@b
    if mode=='bf16': return bf16(a)@bf16(b)
    if mode=='tf32': return tf32(a)@tf32(b)
    if mode=='f16': return f16(a)@f16(b)
    if mode=='bf16x3':
        ah,al=split(a,bf16); bh,bl=split(b,bf16); return ah@bh+ah@bl+al@bh
    if mode=='f16x3':
        ah,al=split(a,f16,2048.); bh,bl=split(b,f16,2048.); return ah@bh+ah@bl+al@bh
    if mode=='bf16x4':
        ah,al=split(a,bf16); bh,bl=split(b,bf16); return ah@bh+ah@bl+al@bh+al@bl
    if mode=='tf32x3':
        ah,al=split(a,tf32); bh,bl=split(b,tf32); return ah@bh+ah@bl+al@bh
    if mode=='bf16x2b':  # second operand (B) in bf16 hi only: Ah Bh + Al Bh
        ah,al=split(a,bf16); bh,_=split(b,bf16); return ah@bh+al@bh
def run(fwd_mode,bwd_mode,rows=1<<16,seed=1):
    cfg=gan.paper_config(param_samples=64,events_per_sample=rows//128,reference_rows=rows,shard_rows=rows//2)
    st=gan.RankState(cfg,0)
    N=cfg.n_events
    rng=np.random.default_rng(seed)
    X=np.concatenate([st.shard[rng.integers(0,cfg.shard_rows,N)], proxy.make_reference(seed+7,[0.9,1.2,0.4,2.1,0.6,0.8],N)])
    t=np.concatenate([np.ones(N),np.zeros(N)])
    Ws,bs=st.dW,st.db; L=len(Ws)
    def forward(mode):
        h=X; cache=[]
        for l in range(L):
            z=(h@Ws[l].T if (l==0 or l==L-1) else mm(h,Ws[l].T,mode))+bs[l]
            cache.append((h,z)); h=mlp.lrelu(z) if l<L-1 else z
        return h[:,0],cache
    z,cache=forward(fwd_mode)
    loss=mlp.bce_with_logits(z,t)
    dz=mlp.bce_grad(z,t)[:,None]
    g=dz; dW=[None]*L
    for l in reversed(range(L)):
        h,zz=cache[l]
        d=g if l==L-1 else g*mlp.lrelu_grad(zz)
        wm,dm=(bwd_mode.split(':')[1].split('/') if bwd_mode.startswith('wg:') else (bwd_mode,bwd_mode))
        if 0<l<L-1: dW[l]=mm(d.T,h,wm); g=mm(d,Ws[l],dm)
        else: dW[l]=d.T@h; g=d@Ws[l]
    return loss,dW
ref_loss,ref_dW=run('f64','f64')
def gerr(a,b):
    fl=1e-2*np.max(np.abs(b)); return np.max(np.abs(a-b)/np.maximum(np.abs(b),fl))
for fm,bm in [('bf16x3','wg:bf16x2b/bf16x3'),('bf16x4','bf16x4'),('bf16x3','bf16x4'),('tf32','tf32'),('bf16','bf16'),('bf16x3','bf16'),('bf16x3','bf16x3'),('f16x3','f16'),('tf32x3','tf32'),('bf16x3','tf32')]:
    l,dW=run(fm,bm)
    print(f"fwd {fm:7s} bwd {bm:7s} loss rel {abs(l-ref_loss)/ref_loss:.2e}  grad max rel(floor1%) {max(gerr(dW[i],ref_dW[i]) for i in range(len(dW))):.2e}")
