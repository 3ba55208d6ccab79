"""Per-CTA timelines of the fused attention kernels (debug hook
dfx_debug_attn_trace; µs from the earliest CTA start):
  --fwd3    persistent forward (default path)
  --kstrip  persistent key-strip backward (default path)
  --bwd     the r01 dq strip kernel (DFX_ATTN_BWD_LEGACY=1)
  (none)    the r01 exact two-pass forward (DFX_ATTN_FWD_LEGACY=1): 0 start,
            1 Q/K landed, 2 softmax ready, 3 S in TMEM, 4 pass-1 done, 5 P
            complete, 6 pass-2 done, 7 O in TMEM, 8 exit."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import _lib  # noqa: E402
from paper_2110_10802_b200 import kernels as K  # noqa: E402

B, S, NH = 8, 512, 12
H = NH * 64
lib = _lib.load()
fn = lib.dfx_debug_attn_trace
fn.argtypes = [ctypes.c_void_p]
qkv = torch.randn(B * S, 3 * H, device="cuda").bfloat16()
am = torch.zeros(B, S, device="cuda")
keep = (torch.rand(B, NH, S, S, device="cuda") > 0.1).to(torch.uint8)
ctx = torch.empty(B * S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, NH, S, device="cuda")
kr = torch.empty(B, NH, S, S // 32, device="cuda", dtype=torch.int32)
kc = torch.empty_like(kr)
if os.environ.get("ATTN_KBIN"):  # packed keep flags as input (the BERT step's mode)
    K.attn_fwd(qkv, B, S, NH, am, keep, 1 / 0.9, 0.125, ctx, lse, kr, kc)
    kr_in = kr.clone()
    run = lambda: K.attn_fwd(qkv, B, S, NH, am, None, 1 / 0.9, 0.125, ctx, lse, kr_in, kc)  # noqa: E731
elif os.environ.get("ATTN_NOKEEP"):  # isolate the dropout-flag traffic
    run = lambda: K.attn_fwd(qkv, B, S, NH, am, None, 1.0, 0.125, ctx, lse, None, None)  # noqa: E731
else:
    run = lambda: K.attn_fwd(qkv, B, S, NH, am, keep, 1 / 0.9, 0.125, ctx, lse, kr, kc)  # noqa: E731
for _ in range(3):
    run()
ncta = B * NH * S // 128
if "--kstrip" in sys.argv:  # persistent key-strip kernel: 0 start, 1 K/V of strip 0, 2-5 S_j of strip 0,
    # 6-8 strip it's gradients done, 10-12 strip it's epilogue done, 15 exit
    run()
    dctx = torch.randn_like(ctx)
    dqkv = torch.empty_like(qkv)
    bwd = lambda: K.attn_bwd(qkv, ctx, dctx, B, S, NH, am, lse, kr, kc, 1 / 0.9, 0.125, dqkv)  # noqa: E731
    for _ in range(3):
        bwd()
    ngrid = min(ncta, torch.cuda.get_device_properties(0).multi_processor_count)
    tr = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
    fn(tr.data_ptr())
    bwd()
    torch.cuda.synchronize()
    fn(None)
    t = tr.view(ncta, 16)[:ngrid].cpu().double()
    rel = (t - t[:, 0].min()) / 1e3
    names = {1: "K/V landed", 2: "S0", 3: "S1", 4: "S2", 5: "S3", 6: "grads0", 10: "epi0", 7: "grads1", 11: "epi1",
             8: "grads2", 12: "epi2", 15: "exit"}
    three = rel[:, 12] > 0
    for lab, m in (("3-strip CTAs", three), ("2-strip CTAs", ~three)):
        r = rel[m]
        print(lab, int(m.sum()), {n: round((r[:, i] - r[:, 0]).mean().item(), 2) for i, n in names.items()
                                  if (r[:, i] > 0).all()})
    print("kernel span", round(rel[:, 15].max().item(), 2), "start spread", round(rel[:, 0].max().item(), 2))
    sys.exit(0)
if "--fwd3" in sys.argv:  # persistent forward: 0 start, 1 Q of strip 0, 2-5 S_j / 6-9 P_j of strip 0,
    # 10-12 strip it's O complete, 15 exit
    ngrid = min(ncta, torch.cuda.get_device_properties(0).multi_processor_count)
    tr = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
    fn(tr.data_ptr())
    run()
    torch.cuda.synchronize()
    fn(None)
    t = tr.view(ncta, 16)[:ngrid].cpu().double()
    rel = (t - t[:, 0].min()) / 1e3
    names = {1: "Q", 2: "S0", 6: "P0", 3: "S1", 7: "P1", 4: "S2", 8: "P2", 5: "S3", 9: "P3", 10: "O0", 11: "O1",
             12: "O2", 15: "exit"}
    three = rel[:, 12] > 0
    for lab, m in (("3-strip CTAs", three), ("2-strip CTAs", ~three)):
        r = rel[m]
        print(lab, int(m.sum()), {n: round((r[:, i] - r[:, 0]).mean().item(), 2) for i, n in names.items()
                                  if (r[:, i] > 0).all()})
    print("kernel span", round(rel[:, 15].max().item(), 2))
    sys.exit(0)
if "--bwd" in sys.argv:  # dq kernel timeline: 0 start, 1 Q/dO landed (MMA), 2-5 S_j ready, 6-9 dS_j done, 10 dQ done, 11 exit
    run()
    dctx = torch.randn_like(ctx)
    dqkv = torch.empty_like(qkv)
    bwd = lambda: K.attn_bwd(qkv, ctx, dctx, B, S, NH, am, lse, kr, kc, 1 / 0.9, 0.125, dqkv)  # noqa: E731
    for _ in range(3):
        bwd()
    tr = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
    fn(tr.data_ptr())
    bwd()
    torch.cuda.synchronize()
    fn(None)
    t = tr.view(ncta, 16).cpu().double()
    rel = (t - t[:, 0].min()) / 1e3
    d = rel[:, 1:12] - rel[:, 0:11]
    names = ["start->qdo", "qdo->S0", "S0->S1", "S1->S2", "S2->S3", "S3->dS0", "dS0->dS1", "dS1->dS2", "dS2->dS3",
             "dS3->dQ", "dQ->exit"]
    print("dq mean phase durations (us):", {n: round(d[:, i].mean().item(), 2) for i, n in enumerate(names)})
    print("dq softmax prologue done (us after start):", round((rel[:, 12] - rel[:, 0]).mean().item(), 2),
          "MMA saw Q/dO:", round((rel[:, 1] - rel[:, 0]).mean().item(), 2))
    print("dq per-CTA total mean", (rel[:, 11] - rel[:, 0]).mean().item(), "kernel span", rel[:, 11].max().item())
    sys.exit(0)
tr = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
fn(tr.data_ptr())
run()
torch.cuda.synchronize()
fn(None)
t = tr.view(ncta, 16).cpu().double()
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print("cta   start   qk   sready  S_in   pass1   P_done  pass2   O_in   exit")
for c in list(range(0, ncta, 37)) + [ncta - 1]:
    print(f"{c:4d} " + " ".join(f"{rel[c, i].item():6.2f}" for i in range(9)))
d = rel[:, 1:9] - rel[:, 0:8]
names = ["setup->qk", "qk->sready", "sready->S", "S->pass1", "pass1->P", "P->pass2", "pass2->O", "O->exit"]
print("mean phase durations (us):", {n: round(d[:, i].mean().item(), 2) for i, n in enumerate(names)})
print("per-CTA total mean", (rel[:, 8] - rel[:, 0]).mean().item(), "kernel span", rel[:, 8].max().item())
