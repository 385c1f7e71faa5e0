import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import torch, math, sys
sys.path.insert(0, '.')
from paper_2509_25191_b200 import ops
def run(D,H,nseq,L, scale=1.0):
    T=nseq*L
    g=torch.Generator(device='cuda').manual_seed(0)
    q,k,v=[(torch.randn(H,T,D,device='cuda',generator=g)*scale).bfloat16() for _ in range(3)]
    o=torch.empty(T,H*D,device='cuda',dtype=torch.bfloat16); lse=torch.empty(H,T,device='cuda')
    ops.attention(q,k,v,o,nseq,L,L,lse=lse)
    qf=q.float().view(H,nseq,L,D); kf=k.float().view(H,nseq,L,D); vf=v.float().view(H,nseq,L,D)
    s=torch.einsum('hsqd,hskd->hsqk',qf,kf)/math.sqrt(D)
    ref=torch.einsum('hsqk,hskd->hsqd',s.softmax(-1),vf).permute(1,2,0,3).reshape(T,H*D)
    lref=torch.logsumexp(s,-1).reshape(H,T)
    err=((o.float()-ref).norm()/ref.norm()).item()
    rowerr=((o.float()-ref).norm(dim=1)/ref.norm(dim=1))
    print(f"D={D} H={H} nseq={nseq} L={L}: rel={err:.3e} lse_maxdiff={(lse-lref).abs().max().item():.3e} worst_rows={rowerr.topk(3).indices.tolist()} {rowerr.max().item():.3e}")
for args in [(64,16,3,1374),(64,1,1,128),(64,1,1,256),(64,2,1,1000),(32,4,8,69),(64,1,1,17)]:
    run(*args)
