"""Prefill (vlc_prefill) against a float64 torch causal attention on a few shapes:
max output error, row max / row sum of the statistics the prefill emits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_23317_b200.prefill import prefill  # noqa: E402


def ref(q, k, v, m):
    B,L,Hq,_,d = q.shape; Hkv = k.shape[2]; G = Hq//Hkv
    qf = q[:,:,:,:m].double(); kf = k[:,:,:,:m].double().repeat_interleave(G, 2); vf = v[:,:,:,:m].double().repeat_interleave(G, 2)
    s = qf @ kf.transpose(-1,-2) / d**0.5
    mask = torch.triu(torch.ones(m, m, dtype=torch.bool, device=q.device), 1)
    s = s.masked_fill(mask, float('-inf'))
    mx = s.max(-1).values
    p = torch.softmax(s, -1)
    return p @ vf, mx, torch.exp(s - mx[..., None]).sum(-1)
for (B,L,Hq,Hkv,d,m,T) in [(1,1,2,1,64,128,128),(1,2,4,2,128,300,310),(1,1,8,2,128,1000,1000),(2,1,4,4,64,77,90)]:
    g = torch.Generator(device='cuda').manual_seed(1)
    q = (torch.randn((B,L,Hq,T,d), device='cuda', generator=g)).to(torch.bfloat16)
    k = torch.randn((B,L,Hkv,T,d), device='cuda', generator=g).to(torch.bfloat16)
    v = torch.randn((B,L,Hkv,T,d), device='cuda', generator=g).to(torch.bfloat16)
    out, rmax, rsum = prefill(q, k, v, m)
    torch.cuda.synchronize()
    o_ref, mx, sm = ref(q, k, v, m)
    err = (out.double() - o_ref).abs().max().item()
    print((B,L,Hq,Hkv,d,m,T), 'out err', err, 'rowmax err', (rmax.double() - mx).abs().max().item(), 'rowsum rel', ((rsum.double()-sm).abs()/sm).max().item(), 'nan', torch.isnan(out).any().item())
