"""One eager EfficientNet-B0 C5 step (batch from EN_N, default 96) after a
warm-up step, between cudaProfilerStart/Stop: the command for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import efficientnet as E  # noqa: E402

N = int(os.environ.get("EN_N", 96))
net = E.EfficientNetB0(E.EffNetConfig(), seed=1)
dev = net.device_inputs(N)
dev["x"].normal_()
dev["labels"].random_(0, 1000)
net.train_step(dev["x"], dev["labels"], 1e-3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
net.train_step(dev["x"], dev["labels"], 1e-3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
