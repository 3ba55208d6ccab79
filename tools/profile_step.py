"""One eager C2 training step (BERT-base layer, bf16, B=8 x S=512) bracketed
by cudaProfilerStart/Stop, for ncu captures of every kernel of the step:

    ncu --set full --clock-control none --import-source on --profile-from-start off \
        -o gpurun_out/step python tools/profile_step.py

(``--workload mbconv`` profiles one C3 MBConv fwd+bwd instead.)  Timing
numbers never come from this script; bench.py measures."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def bert():
    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    B, S, H, NH = 8, 512, 768, 12
    layer = BertEncoderLayer(BertLayerConfig(dtype=torch.bfloat16), device="cuda", seed=1)
    T = B * S
    x = torch.randn(T, H, device="cuda").bfloat16()
    dout = torch.randn(T, H, device="cuda").bfloat16()
    am = torch.zeros(B, S, device="cuda")
    ka = (torch.rand(B, NH, S, S, device="cuda") >= 0.1).to(torch.uint8)
    k1 = (torch.rand(T, H, device="cuda") >= 0.1).to(torch.uint8)
    k2 = (torch.rand(T, H, device="cuda") >= 0.1).to(torch.uint8)

    def step():
        layer.forward(x, am, ka, k1, k2)
        layer.backward(dout)
        layer.sgd_step(1e-4)

    return step


def mbconv():
    from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig

    N, HW, C = 96, 112, 96
    blk = MBConvBlock(MBConvConfig(channels=C, dtype=torch.bfloat16), device="cuda", seed=1)
    x = torch.randn(N, HW, HW, C, device="cuda").bfloat16()
    dy = torch.randn(N, HW, HW, C, device="cuda").bfloat16()

    def step():
        blk.forward(x)
        blk.backward(dy)

    return step


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", choices=["bert", "mbconv"], default="bert")
    a = ap.parse_args()
    step = bert() if a.workload == "bert" else mbconv()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
