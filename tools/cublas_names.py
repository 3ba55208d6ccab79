import torch
from torch.profiler import profile, ProfilerActivity
T,H,F=4096,768,3072
cases=[("ffn1",T,F,H),("ffn2",T,H,F),("qkv",T,3*H,H),("out",T,H,H)]
for name,m,n,k in cases:
    a=torch.randn(m,k,device="cuda").bfloat16(); b=torch.randn(n,k,device="cuda").bfloat16()
    for _ in range(3): torch.matmul(a,b.t())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.matmul(a,b.t()); torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type.name=="CUDA": print(name, e.name[:200])
