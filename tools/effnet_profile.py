"""Per-call-site time of the EfficientNet-B0 C5 step (batch 96, 224x224,
bf16): every library call labelled with its block, top rows by time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import efficientnet as E  # noqa: E402
from paper_2110_10802_b200 import kernels as K  # noqa: E402
from paper_2110_10802_b200.graphs import CapturedStep  # noqa: E402

N = int(os.environ.get("EN_N", 96))
net = E.EfficientNetB0(E.EffNetConfig(), seed=1)
dev = net.device_inputs(N)
dev["x"].normal_()
dev["labels"].random_(0, 1000)
for i, b in enumerate(net.blocks):  # label every call with its block
    for nm in ("forward", "backward"):
        f = getattr(b, nm)

        def wrap(*a, _f=f, _i=i, _nm=nm, **kw):
            with K.label(f"b{_i}.{_nm}"):
                return _f(*a, **kw)
        setattr(b, nm, wrap)
K._LABEL_NEST = True  # noqa: used by kernels._span
timer = K.KernelTimer()
fn = lambda: net.train_step(dev["x"], dev["labels"], 1e-3)  # noqa: E731
cs = CapturedStep(fn)
with timer:
    inst = CapturedStep(fn, warmup=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(5):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cs.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"C5 step {sorted(ts)[2]:.3f} ms  ({N * 1e3 / sorted(ts)[2]:.0f} img/s)")
timer.totals = {}
for _ in range(3):
    flush.zero_()
    inst.replay()
    timer.collect()
rows = timer.summary()
tot = sum(r["ms"] for r in rows)
print(f"instrumented sum {tot / 3:.3f} ms")
for r in rows[:45]:
    ms = r["ms"] / 3
    rate = r["work"] / 3 / (ms * 1e-3)
    unit = "GB/s" if r["kind"] == "hbm" else "TF/s"
    rate = rate / 1e9 if unit == "GB/s" else rate / 1e12
    print(f"{r['label']:40s} {ms * 1e3:8.1f} us {100 * r['ms'] / tot:5.1f}% {rate:8.1f} {unit}")
agg = {}
for r in rows:
    k = r["label"].split("/", 1)[-1] if "/" in r["label"] else r["label"]
    a = agg.setdefault(k, [0.0, 0])
    a[0] += r["ms"] / 3
    a[1] += 1
print("---- by kernel type")
for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:40s} {ms * 1e3:8.1f} us  {100 * ms * 3 / tot:5.1f}%  ({n} sites)")
