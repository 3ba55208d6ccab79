"""CUDA-event timing of the fused attention kernels at the C2 shape (B=8, S=512,
12 heads): forward with unpacked keep flags, forward with packed keep input (the
BERT step's mode), and the backward. Prints mean µs per launch (CUDA-graph replay)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402

B, S, NH = 8, 512, 12
H = NH * 64
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(B * S, 3 * H, device="cuda", generator=g).bfloat16()
am = torch.zeros(B, S, device="cuda")
keep = (torch.rand(B, NH, S, S, device="cuda", generator=g) > 0.1).to(torch.uint8)
ctx = torch.empty(B * S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, NH, S, device="cuda")
kr = torch.empty(B, NH, S, S // 32, device="cuda", dtype=torch.int32)
kc = torch.empty_like(kr)
K.attn_fwd(qkv, B, S, NH, am, keep, 1 / 0.9, 0.125, ctx, lse, kr, kc)  # makes the packed flags
kr_in = kr.clone()
dctx = torch.randn(ctx.shape, device="cuda", generator=g).bfloat16()
dqkv = torch.empty_like(qkv)


def timeit(fn, n=20, reps=5):
    """Mean µs per launch of n launches captured in one CUDA graph (no host
    launch overhead in the measurement)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n * reps) * 1e3


if os.environ.get("ATTN_ONLY") == "packed":  # one packed-keep forward + backward (for ncu)
    K.attn_fwd(qkv, B, S, NH, am, None, 1 / 0.9, 0.125, ctx, lse, kr_in, kc)
    K.attn_bwd(qkv, ctx, dctx, B, S, NH, am, lse, kr_in, kc, 1 / 0.9, 0.125, dqkv)
    torch.cuda.synchronize()
    sys.exit(0)
print("fwd u8 keep   us", round(timeit(lambda: K.attn_fwd(qkv, B, S, NH, am, keep, 1 / 0.9, 0.125, ctx, lse, kr, kc)), 2))
print("fwd packed in us", round(timeit(lambda: K.attn_fwd(qkv, B, S, NH, am, None, 1 / 0.9, 0.125, ctx, lse, kr_in, kc)), 2))
print("bwd           us", round(timeit(lambda: K.attn_bwd(qkv, ctx, dctx, B, S, NH, am, lse, kr_in, kc, 1 / 0.9, 0.125,
                                                            dqkv)), 2))
