"""Benchmark of the fused training hot path (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one training step of a BERT-base encoder layer (H=768, 12 heads,
FFN 3072, post-LN, tanh-GELU, dropout p=0.1 with explicit keep masks) in bf16
at batch 8 x seq 512 per GPU: forward + backward + SGD update (+ gradient
allreduce over NCCL when N > 1, weak scaling).  Synthetic inputs and
random-init weights (seeded), resident in HBM for ``value``; ``e2e`` repeats
the measurement through the host-buffer API (pinned H2D of the step's inputs,
D2H of dx inside the timed region).

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launching stream, with a 256 MiB L2 flush between steps (outside the events);
barrier + synchronize on both sides; max over ranks.  Every library call is
also bracketed by events to attribute time per kernel; the dominant one is
reported against MEASURED_PEAKS.json as ``roofline``.

``--impl reference`` times the reference itself — the ``dfir`` package
installed from /root/reference into baseline/_ref (git-ignored, travels to the
GPU box) — on this host: ``interp.execute`` of the reference's own BERT-layer
graph (oracle/make_golden.bert_layer_model) forward +
``differentiate_graph`` backward, one sequence (B=1, S=512) per step
(BASELINE.md §2).  The float64 numpy port (oracle/oracle.py) is reported
beside it as a second reading.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, S, H, NH, FF = 8, 512, 768, 12, 3072
P_DROP = 0.1
METRIC = "BERT-base encoder layer fwd+bwd+SGD training throughput (bf16, B=8 x S=512 per GPU)"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 / C5 workload measurements")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU reference path (oracle port, float64 numpy — the reference computes in f64)


def cpu_reference_sample(seconds: float, seq=S):
    """Run fwd+bwd of ONE sequence (B=1, S=512) through the oracle until
    ``seconds`` have elapsed (at least once).  Returns (samples/s, reps)."""
    import numpy as np

    from oracle import oracle as O

    rng = np.random.default_rng(0)
    T = seq
    prm = {}
    for nm, shp in [("wq", (H, H)), ("wk", (H, H)), ("wv", (H, H)), ("wo", (H, H)),
                    ("w1", (FF, H)), ("w2", (H, FF))]:
        prm[nm] = 0.02 * rng.standard_normal(shp)
    for nm, n in [("bq", H), ("bk", H), ("bv", H), ("bo", H), ("b1", FF), ("b2", H)]:
        prm[nm] = 0.1 * rng.standard_normal(n)
    for i in "12":
        prm["g" + i] = 1 + 0.1 * rng.standard_normal(H)
        prm["be" + i] = 0.1 * rng.standard_normal(H)
    x = rng.standard_normal((T, H))
    am = np.zeros((1, 1, 1, seq))
    dm = O.mask_values(rng.random((1, NH, seq, seq)) >= P_DROP, P_DROP, np.float64)
    m1 = O.mask_values(rng.random((T, H)) >= P_DROP, P_DROP, np.float64)
    m2 = O.mask_values(rng.random((T, H)) >= P_DROP, P_DROP, np.float64)
    dout = rng.standard_normal((T, H))
    reps = 0
    t0 = time.perf_counter()
    while True:
        out, cache = O.bert_layer_fwd(prm, x, am, dm, m1, m2, 1, seq, NH, 1e-12)
        O.bert_layer_bwd(prm, cache, dout)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return reps / el, reps, el


class DfirReference:
    """The reference package itself (dfir, baseline/_ref): the BERT-layer graph
    of registry operators imported, differentiated once
    (graph construction, not timed), then one ``interp.execute`` of the forward
    + backward states per step on one sequence."""

    def __init__(self, seq=S):
        import numpy as np

        ref = os.path.join(ROOT, "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "dfir")):
            raise ImportError("reference dfir package not installed in baseline/_ref")
        if ref not in sys.path:
            sys.path.insert(0, ref)
        from dfir import autodiff, frontend, interp

        from oracle import make_golden as mg  # graph builder only (registry ops, no arithmetic)

        self.interp = interp
        doc, out, wnames = mg.bert_layer_model(1, seq, H, NH, FF, 1e-12, "f32")
        rng = np.random.default_rng(0)
        inputs, _ = mg.bert_layer_inputs(rng, 1, seq, H, NH, FF, P_DROP, np.float32)
        t0 = time.perf_counter()
        g = frontend.import_model(doc)
        res = autodiff.differentiate_graph(
            g, autodiff.GradientRequest(outputs=(out,), wrt=tuple(["x"] + wnames), seed="input"))
        self.ad_s = time.perf_counter() - t0
        self.graph = res.graph
        self.inputs = dict(inputs)
        self.inputs[res.adjoints.grads[out]] = rng.standard_normal((seq, H)).astype(np.float32)

    def step(self):
        t0 = time.perf_counter()
        self.interp.execute(self.graph, self.inputs)
        return time.perf_counter() - t0


_T0 = time.time()


def _progress(what):
    """stderr breadcrumbs (the JSON line alone goes to stdout)."""
    print(f"[bench {time.time() - _T0:7.1f} s] {what}", file=sys.stderr, flush=True)


def reference_sample(seconds: float):
    """Bounded cpu_baseline reading: the reference package (``kind``
    "reference") when installed, else the numpy port.  Returns
    (samples/s, sample text, kind)."""
    try:
        ref = DfirReference()
    except ImportError:
        v, reps, el = cpu_reference_sample(seconds)
        return v, f"{reps} x one sequence (B=1, S={S}) fwd+bwd, float64 numpy port (oracle/oracle.py), {el:.1f} s", \
            "port"
    t, reps = 0.0, 0
    while t < seconds or reps == 0:
        t += ref.step()
        reps += 1
    return reps / t, (f"{reps} x one sequence (B=1, S={S}) fwd+bwd through dfir interp.execute "
                      f"(reference package, baseline/_ref), {t:.1f} s"), "reference"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count()
    budget = 150.0  # seconds of timed reference work (the whole run stays within a few minutes)
    try:
        ref = DfirReference()
        kind = "reference"
        step = ref.step
    except ImportError:
        ref, kind = None, "port"

        def step():
            return cpu_reference_sample(0.0)[2]
    warm = 0
    t_w = 0.0
    for _ in range(max(args.warmup, 1)):
        t_w += step()
        warm += 1
        if t_w > 30:
            break
    per_step = []
    for _ in range(args.steps):
        per_step.append(step())
        if sum(per_step) > budget:
            break
    k = len(per_step)
    ms = 1e3 * statistics.median(per_step)
    value = 1e3 / ms  # one sequence per step
    if kind == "reference":
        sample = (f"1 sequence (B=1, S={S}) fwd+bwd per step through the reference package: dfir "
                  f"interp.execute of differentiate_graph(bert_layer_model) (baseline/_ref), f32 graph "
                  f"(f64 arithmetic inside reference_apply), median of {k} steps; graph AD once "
                  f"({ref.ad_s:.2f} s, untimed)")
    else:
        sample = f"1 sequence (B=1, S={S}) fwd+bwd per step, float64 numpy port (oracle/oracle.py), {k} steps"
    port_v, _, port_el = cpu_reference_sample(10.0) if kind == "reference" else (None, 0, 0)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": k, "warmup": warm, "ms_per_step": round(ms, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy)",
        "config": {"workload": "bert_base_encoder_layer_train_step (BASELINE.json configs[1]); bounded sample: "
                               "one sequence per step", "global_batch": 1, "seq_len": S,
                   "hidden": H, "heads": NH, "ffn": FF, "parallelism": "cpu",
                   "same_config": False, "why": "B=8 x S=512 takes ~25 s per step in the reference; samples/s "
                                                "normalises the bounded one-sequence sample"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")},
        "port_reading": None if port_v is None else {
            "value": round(port_v, 4), "unit": UNIT, "kind": "port",
            "sample": f"float64 numpy restatement (oracle/oracle.py), {port_el:.1f} s"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clock / power / throttle-reason samples taken DURING the timed
    region by a background thread polling NVML every 5 ms (nvidia-smi's
    100 ms loop sees at most a sample or two of a sub-second timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index, period_s=0.005):
        self.index, self.period = index, period_s
        self.rows, self.thread, self.nv = [], None, None

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 — no NVML: report "unsampled"
            self.nv = None
            return self
        self.stop = threading.Event()
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()
        return self

    def _loop(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetPowerUsage(h) / 1e3,
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h),
                                  nv.nvmlDeviceGetUtilizationRates(h).gpu))
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(self.period)

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        busy = [r for r in self.rows if r[3] > 0] or self.rows
        reasons = sorted({n for r in busy for n, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(busy),
                "power_w_max": round(max(r[1] for r in self.rows), 1), "source": "NVML, 5 ms poll"}


# ---------------------------------------------------------------------------
# our path


def peaks(clocks=None):
    """Roofline denominators.  Tensor: the measured BURST cuBLAS figure when the
    timed region ran uncapped at max clocks (no sw_power_cap, median SM clock
    >= 95 % of max), else the sustained (power-capped) figure."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        pk = {"hbm_gbs": d["hbm_gbs"], "tflops_burst": d["bf16_tflops"],
              "tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
              "source": "measured (MEASURED_PEAKS.json)"}
    else:
        pk = {"hbm_gbs": 6650.0, "tflops_burst": 1590.0, "tflops_sustained": 1590.0,
              "source": "fallback (B200_PROFILING.md)"}
    capped = True
    if clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz"):
        capped = "sw_power_cap" in clocks["reasons"] or clocks["sm_mhz"] < 0.95 * clocks["sm_max_mhz"]
    pk["tflops"] = pk["tflops_sustained"] if capped else pk["tflops_burst"]
    pk["tensor_peak"] = "sustained (power cap / clocks below max in the timed region)" if capped else \
        "burst (uncapped, SM clock at max in the timed region)"
    return pk


def _kernel_rows(timer, steps, pk):
    """Per call-site rows.  A contraction whose arithmetic intensity (flops per
    compulsory operand byte) is below the ridge point peak_flops / peak_HBM is
    HBM-bound and is reported in GB/s against HBM (e.g. EfficientNet's 1x1
    convolutions with K = 16..192)."""
    ridge = pk["tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    rows = []
    for r in timer.summary():
        per_call_ms = r["ms"] / r["calls"]
        work = r["work"] / r["calls"]
        nbytes = r.get("bytes", 0.0) / r["calls"]
        row = {"kernel": r["label"], "calls_per_step": r["calls"] / steps, "us_per_call": round(per_call_ms * 1e3, 2),
               "share": 0.0}
        if r["kind"] != "hbm" and nbytes > 0 and work / nbytes < ridge:
            row["flops_per_byte"] = round(work / nbytes, 1)
            row["tflops"] = round(work / (per_call_ms * 1e-3) / 1e12, 1)
            kind, work = "hbm", nbytes
        else:
            kind = r["kind"]
        if kind == "hbm":
            ach, peak, unit = work / (per_call_ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
        else:
            ach, peak, unit = work / (per_call_ms * 1e-3) / 1e12, pk["tflops"], "TFLOP/s"
        row.update({"bound": "hbm" if kind == "hbm" else "tensor", "achieved": round(ach, 1), "unit": unit,
                    "frac": round(ach / peak, 3), "work_per_call": work})
        rows.append(row)
    tot = sum(r["us_per_call"] * r["calls_per_step"] for r in rows) or 1.0
    for r in rows:
        r["share"] = round(r["us_per_call"] * r["calls_per_step"] / tot, 3)
    rows.sort(key=lambda r: -r["share"])
    return rows


def _timed_graph(step, k, flush):
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    torch.cuda.synchronize()
    for i in range(k):
        flush.zero_()
        evs[i][0].record()
        step()
        evs[i][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / k


def measure_bert_c1(steps, flush, pk):
    """BASELINE.json configs[0]: one BERT-base encoder layer, fp32, B=2 x S=128,
    fwd + bwd + SGD (the reference's CPU-oracle workload; CUDA-core fp32 GEMMs
    for the 1e-4 parity bar) as a CUDA graph, next to the oracle on the host."""
    import torch

    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    b1, s1 = 2, 128
    layer = BertEncoderLayer(BertLayerConfig(dtype=torch.float32), device="cuda", seed=3)
    g = torch.Generator(device="cpu").manual_seed(5)
    dev = layer.device_inputs(b1, s1)
    dev["x"].copy_(torch.randn(b1 * s1, H, generator=g))
    dev["dout"].copy_(torch.randn(b1 * s1, H, generator=g))
    dev["add_mask"].zero_()
    for k in ("keep_attn", "keep1", "keep2"):
        dev[k].copy_((torch.rand(dev[k].shape, generator=g) >= P_DROP).to(dev[k].dtype))
    cs = layer.capture_step(b1, s1, 1e-4)
    ms = _timed_graph(cs.replay, steps, flush)
    v, reps, el = cpu_reference_sample(3.0, seq=s1)
    return {"metric": "BERT-base encoder layer fwd+bwd+SGD, fp32, B=2 x S=128 (C1)",
            "value": round(b1 * 1e3 / ms, 1), "unit": "samples/s", "ms_per_step": round(ms, 4),
            "config": {"workload": "bert_base_encoder_layer_train_step fp32 (BASELINE.json configs[0])",
                       "global_batch": b1, "seq_len": s1, "dtype": "f32"},
            "cpu_oracle": {"value": round(v * 1.0, 3), "unit": "samples/s", "sample": f"{reps} x one sequence S={s1}",
                           "cores": os.cpu_count()},
            "note": "launch-bound: every kernel moves 1-5 MB (SURVEY.md §7 hard parts)"}


def measure_norm_sweep_c4(steps, flush, pk):
    """BASELINE.json configs[3]: LayerNorm vs BatchNorm (+ swish) over the
    channel axis of channels-last 4D [32,56,56,64] and 5D [8,16,56,56,32]
    bf16 tensors, fwd + bwd each; effective HBM GB/s over the compulsory
    passes (LN: fwd read x + write y, bwd read dy, x + write dx; BN: fwd 2 reads
    + 1 write, bwd 3 reads + 1 write)."""
    import torch

    from paper_2110_10802_b200.graphs import CapturedStep
    from paper_2110_10802_b200.norms import BatchNormAct, LayerNormAct

    out = {}
    for name, shape in (("4d", (32, 56, 56, 64)), ("5d", (8, 16, 56, 56, 32))):
        C = shape[-1]
        g = torch.Generator(device="cpu").manual_seed(9)
        x = torch.randn(shape, generator=g).bfloat16().cuda()
        dy = torch.randn(shape, generator=g).bfloat16().cuda()
        n = x.numel() * 2
        for kind, mod, passes in (("layernorm_swish", LayerNormAct(C, act="swish"), 5),
                                  ("batchnorm_swish", BatchNormAct(C, act="swish"), 7)):
            def fn(m=mod):
                m.forward(x)
                m.backward(dy)

            cs = CapturedStep(fn)
            ms = _timed_graph(cs.replay, steps, flush)
            gbs = passes * n / (ms * 1e-3) / 1e9
            out[f"{kind}_{name}"] = {"shape": list(shape), "us_fwd_bwd": round(ms * 1e3, 2),
                                     "hbm_gbs_effective": round(gbs, 1),
                                     "hbm_frac_effective": round(gbs / pk["hbm_gbs"], 3)}
    return {"metric": "normalisation sweep fwd+bwd (LN vs BN + swish, channels-last bf16) (C4)",
            "config": {"workload": "norm_sweep (BASELINE.json configs[3])"}, "cases": out}


def _mbconv_vs_unfused(ours):
    path = os.path.join(ROOT, "tests", "golden", "movement_volume.json")
    if not os.path.exists(path):
        return None
    ref = json.load(open(path))["mbconv_c3"]["fwd_bwd_library_bytes"] / 2
    return {"ours_bytes_per_step": ours, "reference_unfused_bytes_per_step_bf16": int(ref),
            "ratio": round(ours / ref, 4)}


def measure_mbconv_c3(steps, flush, pk):
    """BASELINE.json configs[2]: one MBConv block (dw3x3 + BN + swish + SE),
    N=96 x 112x112 x 96 channels, bf16, fwd + bwd as a CUDA graph."""
    import torch

    from paper_2110_10802_b200 import kernels as K
    from paper_2110_10802_b200.graphs import CapturedStep
    from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig

    N, HW, C = 96, 112, 96
    blk = MBConvBlock(MBConvConfig(channels=C, dtype=torch.bfloat16), device="cuda", seed=1)
    g = torch.Generator(device="cpu").manual_seed(7)
    x = torch.randn(N, HW, HW, C, generator=g).bfloat16().cuda()
    dy = torch.randn(N, HW, HW, C, generator=g).bfloat16().cuda()

    def fn():
        blk.forward(x)
        blk.backward(dy)

    cs = CapturedStep(fn)
    timer = K.KernelTimer()
    with timer:
        inst = CapturedStep(fn, warmup=0)
    ms = _timed_graph(cs.replay, steps, flush)
    timer.totals = {}
    for _ in range(max(3, steps // 4)):
        flush.zero_()
        inst.replay()
        timer.collect()
    rows = _kernel_rows(timer, max(3, steps // 4), pk)
    elems = N * HW * HW * C
    # compulsory traffic of the schedule: fwd conv (x, z) + pool (z) + excite (z, y);
    # bwd reduce (dy, z) + dz/dw (x, dy, z, dz) + dx (dz, dx) = 13 tensor passes
    traffic = 13 * elems * 2
    return {"metric": "MBConv block fwd+bwd throughput (bf16, N=96, 112x112, C=96, dw3x3+BN+swish+SE)",
            "value": round(N * 1e3 / ms, 1), "unit": "images/s", "ms_per_step": round(ms, 4),
            "config": {"workload": "mbconv_block (BASELINE.json configs[2])", "batch": N, "hw": HW,
                       "channels": C, "stride": 1, "se": 4, "dtype": "bf16"},
            "hbm_gbs_effective": round(traffic / (ms * 1e-3) / 1e9, 1),
            "bytes_vs_unfused": _mbconv_vs_unfused(traffic),
            "hbm_frac_effective": round(traffic / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 3),
            "kernels": rows[:10]}


def measure_effnet_c5(steps, flush, pk, world, rank, local, dist):
    """BASELINE.json configs[4]: full EfficientNet-B0 training step, 96 images
    of 224x224 per GPU, SyncBN + gradient allreduce when world > 1."""
    import torch

    from paper_2110_10802_b200 import kernels as K
    from paper_2110_10802_b200.efficientnet import EfficientNetB0, EffNetConfig

    N = 96
    pg = dist.group.WORLD if world > 1 else None
    net = EfficientNetB0(EffNetConfig(), device=f"cuda:{local}", seed=11, process_group=pg)
    g = torch.Generator(device="cpu").manual_seed(200 + rank)
    xh = torch.randn(N, 224, 224, 3, generator=g).bfloat16().pin_memory()
    lh = torch.randint(0, 1000, (N,), generator=g, dtype=torch.int32).pin_memory()
    dev = net.device_inputs(N)
    dev["x"].copy_(xh)
    dev["labels"].copy_(lh)
    lr = 1e-3
    rows = []
    from paper_2110_10802_b200.graphs import CapturedStep

    # one CUDA graph per step; data parallel, the SyncBN statistics
    # collectives and the group-aligned gradient buckets are NCCL nodes of it
    cs = net.capture_step(N, lr)
    step = cs.replay
    if world == 1:
        timer = K.KernelTimer()
        net.concurrent = False  # single-stream twin: per-kernel times without branch contention
        with timer:
            inst = CapturedStep(lambda: net.train_step(dev["x"], dev["labels"], lr), warmup=0)
        net.concurrent = True
        timer.totals = {}
        for _ in range(3):
            flush.zero_()
            inst.replay()
            timer.collect()
        rows = _kernel_rows(timer, 3, pk)
    for _ in range(3):
        step()
    if world > 1:
        dist.barrier()
    ms = _timed_graph(step, steps, flush)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    loss_h = torch.empty(1).pin_memory()
    ke = max(3, steps // 2)
    if world == 1:  # pipelined: step i+1's H2D and step i's D2H overlap step i
        for _ in range(3):
            net.train_step_host_async(xh, lh, lr=lr, loss_host=loss_h)
        net.finish_host()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ke):
            net.train_step_host_async(xh, lh, lr=lr, loss_host=loss_h)
        net.finish_host()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / ke
    else:
        def host_step():
            net.train_step_host(xh, lh, lr=lr, loss_host=loss_h, graph=cs)

        e2e_ms = _timed_graph(host_step, ke, flush)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d, d2h = net.host_inputs_bytes(N)
    return {"metric": "EfficientNet-B0 training step throughput (bf16, 96 images/GPU, 224x224)",
            "value": round(world * N * 1e3 / ms, 1), "unit": "images/s", "ms_per_step": round(ms, 3),
            "n_gpus": world, "scaling": "weak",
            "config": {"workload": "efficientnet_b0_train_step (BASELINE.json configs[4])", "batch_per_gpu": N,
                       "image": 224, "params": net.num_params, "parallelism": f"dp{world}",
                       "syncbn": world > 1, "step": "fwd + bwd + SGD" + (" + bucketed NCCL allreduce" if world > 1 else ""),
                       "execution": "CUDA graph" + (" (SyncBN + gradient buckets as NCCL nodes)" if world > 1 else "")},
            "e2e": {"value": round(world * N * 1e3 / e2e_ms, 1), "unit": "images/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "kernels": rows[:12]}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2110_10802_b200 import kernels as K
    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    cfg = BertLayerConfig(hidden=H, heads=NH, ffn=FF, p_drop=P_DROP, dtype=torch.bfloat16)
    layer = BertEncoderLayer(cfg, device=f"cuda:{local}", seed=1234)
    T = B * S
    gen = torch.Generator(device="cpu").manual_seed(100 + rank)
    x = torch.randn(T, H, generator=gen).bfloat16()
    dout = torch.randn(T, H, generator=gen).bfloat16()
    am = torch.where(torch.rand(B, S, generator=gen) < 0.1, -10000.0, 0.0).float()
    keep_attn = (torch.rand(B, NH, S, S, generator=gen) >= P_DROP).to(torch.uint8)
    keep1 = (torch.rand(T, H, generator=gen) >= P_DROP).to(torch.uint8)
    keep2 = (torch.rand(T, H, generator=gen) >= P_DROP).to(torch.uint8)
    # the attention dropout mask is supplied bit-packed (the fused kernels' native
    # form: 3.1 MB instead of 25 MB of u8 flags per step over PCIe and HBM)
    keep_attn_bits = K.pack_keep_bits(keep_attn)
    # ... and so are the two BDRLN dropout masks (0.4 MB each instead of 3.1 MB)
    host = {k: v.pin_memory() for k, v in dict(x=x, dout=dout, add_mask=am, keep_attn=keep_attn_bits,
                                                 keep1=K.pack_keep_bits(keep1),
                                                 keep2=K.pack_keep_bits(keep2)).items()}
    dev = layer.device_inputs(B, S)
    for k, v in host.items():
        dev[k].copy_(v)
    dx_host = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    lr = 1e-4
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # The step is captured once into a CUDA graph (host launch path off the
    # critical path); an instrumented twin with event-record nodes around
    # every library call attributes time per kernel in a second pass.
    K.reset_launch_count()
    timer = K.KernelTimer()
    if world > 1:
        # data parallel: the backward all-reduces the gradient arena in four
        # group-aligned buckets as the groups complete (overlapping the rest
        # of the backward); the buckets are NCCL nodes of the step's graph
        layer.attach_process_group(dist.group.WORLD)
    g_step, g_inst = layer.capture_step(B, S, lr, timer)
    K.reset_launch_count()  # count one eager step's launches (the graph replays the same set)
    saved = [t.clone() for t in layer.training_state()]
    layer.train_step(dev["x"], dev["add_mask"], dev["keep_attn"], dev["keep1"], dev["keep2"], dev["dout"], lr)
    for t, v in zip(layer.training_state(), saved):
        t.copy_(v)
    launches_per_step = K.launch_count()

    def step(g=g_step):
        g.replay()

    def timed(fn, k, per_step=None):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(k):
            flush.zero_()
            evs[i][0].record()
            fn()
            evs[i][1].record()
            if per_step is not None:
                per_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    _progress("bert c2 captured; timing")
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(max(3, args.warmup)):
            step()
        torch.cuda.synchronize()
        total_ms = timed(step, args.steps)
        launches = launches_per_step * args.steps
        # attribution pass: same step with event-record nodes, collected per replay
        timer.totals = {}
        inst_ms = timed(lambda: step(g_inst), args.steps, per_step=timer.collect)
    clocks = sampler.summary()
    ms_step = total_ms / args.steps
    value = world * B * 1e3 / ms_step

    # e2e through the host-buffer API (pinned H2D of inputs, graph replay, D2H of dx).
    # N=1: the pipelined form (two input/activation sets; step i+1's H2D and
    # step i's D2H overlap step i's compute), timed as ONE region from the
    # first H2D to the last dx landing on the host, divided by the step count.
    ke = max(5, args.steps // 2)
    if world == 1:
        for _ in range(3):
            layer.train_step_host_async(host, lr=lr, dx_host=dx_host)
        layer.finish_host()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ke):
            layer.train_step_host_async(host, lr=lr, dx_host=dx_host)
        layer.finish_host()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / ke
    else:
        def host_step():  # captured step (gradient buckets inside) from host buffers
            layer.train_step_host(host, lr=lr, dx_host=dx_host)

        for _ in range(3):
            host_step()
        e2e_ms = timed(host_step, ke) / ke
    h2d, d2h = layer.host_inputs_bytes(B, S)

    # per-kernel roofline (tensor denominator chosen from the clocks sampled above)
    pk = peaks(clocks)
    rows = _kernel_rows(timer, args.steps, pk)
    dom = max(rows, key=lambda r: r["us_per_call"] * r["calls_per_step"])
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set
    # full capture (profiles/r01_traffic.json, tools/gpu_profile.sh); null if absent
    traffic = None
    tsrc = None
    for tname in ("r02_traffic.json", "r01_traffic.json"):  # newest capture first
        tpath = os.path.join(ROOT, "profiles", tname)
        if os.path.exists(tpath) and dom["kernel"] in json.load(open(tpath)):
            traffic, tsrc = json.load(open(tpath))[dom["kernel"]], f"profiles/{tname} (ncu DRAM bytes)"
            break
    roofline = {"bound": dom["bound"], "kernel": dom["kernel"], "achieved": dom["achieved"],
                "peak": pk["hbm_gbs"] if dom["bound"] == "hbm" else pk["tflops"], "unit": dom["unit"],
                "frac": dom["frac"], "traffic": traffic, "traffic_source": tsrc,
                "peak_source": pk["source"] + (", tensor " + pk["tensor_peak"] if dom["bound"] == "tensor" else "")}
    gemm_us = sum(r["us_per_call"] * r["calls_per_step"] for r in rows if r["bound"] == "tensor")
    flops = layer.step_flops(B, S)
    gemm_tflops = flops / (gemm_us * 1e-6) / 1e12

    workloads = {}
    if not args.no_extra:
        if rank == 0 and world == 1:
            _progress("bert_c1_fp32")
            workloads["bert_c1_fp32"] = measure_bert_c1(max(10, args.steps // 4), flush, pk)
            _progress("mbconv_c3")
            workloads["mbconv_c3"] = measure_mbconv_c3(max(10, args.steps // 4), flush, pk)
            _progress("norm_sweep_c4")
            workloads["norm_sweep_c4"] = measure_norm_sweep_c4(max(10, args.steps // 4), flush, pk)
        _progress("efficientnet_b0_c5")
        workloads["efficientnet_b0_c5"] = measure_effnet_c5(max(5, args.steps // 20), flush, pk, world, rank,
                                                            local, dist)
        _progress("workloads done")

    # the fused schedule's compulsory bytes vs the reference's unfused graph
    # (ir.movement_volume of the autodiff graph, oracle/movement_volume.py; f32 -> bf16 halved)
    mv_path = os.path.join(ROOT, "tests", "golden", "movement_volume.json")
    bytes_vs_unfused = None
    if os.path.exists(mv_path):
        mv = json.load(open(mv_path))
        ref_b = mv["bert_c2"]["fwd_bwd_library_bytes"] / 2
        ours_b = layer.step_bytes(B, S)
        bytes_vs_unfused = {"ours_bytes_per_step": ours_b, "reference_unfused_bytes_per_step_bf16": int(ref_b),
                            "ratio": round(ours_b / ref_b, 4),
                            "reference": "dfir ir.movement_volume of differentiate_graph(BERT layer) "
                                         "(library-node form, f32 halved to bf16)",
                            "achieved_gbs": round(ours_b / (ms_step * 1e-3) / 1e9, 1)}

    cpu = None
    _progress("cpu baseline")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample, kind = reference_sample(args.cpu_seconds)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": os.cpu_count(), "kind": kind, "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded torch.randn inputs, random-init weights, explicit dropout keep masks)",
            "config": {"workload": "bert_base_encoder_layer_train_step (BASELINE.json configs[1])",
                       "global_batch": B * world, "seq_len": S, "hidden": H, "heads": NH, "ffn": FF,
                       "parallelism": f"dp{world}", "l2": "flushed (256 MiB write) between timed steps",
                       "step": "fwd + bwd + SGD" + (" + NCCL grad allreduce" if world > 1 else "")},
            "e2e": {"value": round(world * B * 1e3 / e2e_ms, 2), "unit": UNIT, "ms_per_step": round(e2e_ms, 4),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "instrumented_ms_per_step": round(inst_ms / args.steps, 4),
            "roofline": roofline,
            "gemm_tflops": round(gemm_tflops, 1),
            "kernels": rows,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "workloads": workloads,
            "bytes_vs_unfused": bytes_vs_unfused,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
