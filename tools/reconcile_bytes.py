"""Reconcile the HBM traffic of one fused BERT C2 training step three ways
(SURVEY.md §8 a14 / §8f row 4):

  measured   sum over the step's launches of ncu dram__bytes_read.sum +
             dram__bytes_write.sum (one replay of the captured step, cold L2:
             bench.py flushes L2 before every step);
  schedule   BertEncoderLayer.step_bytes(B, S): every kernel's tensor
             arguments read once + written once (bench.py's "ours" side);
  reference  dfir ir.movement_volume (ir.py:790-835) of the reference's unfused
             forward+backward graph (tests/golden/movement_volume.json, f32,
             halved for bf16).

Input: an ncu CSV captured with
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      --clock-control none --csv --log-file X.csv python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline
The step is the launches after the last L2-flush fill (torch FillFunctor) of the
uninstrumented replays, i.e. the block before the instrumented twin starts
(the twin's launches are identical; either block may be used, --block picks).

Prints a markdown table (per launch and totals) and exits non-zero when the
measured bytes exceed the schedule's compulsory bytes by more than --slack.
"""

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B, S = 8, 512


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = {}
    order = []
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        if key not in launches:
            launches[key] = {"name": d["Kernel Name"], "grid": d.get("Grid Size", "")}
            order.append(key)
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        launches[key][d["Metric Name"]] = v * scale
    return [launches[k] for k in order]


def steps(launches):
    """Blocks of launches between L2-flush fills."""
    out, cur = [], []
    for d in launches:
        if "FillFunctor" in d["name"]:
            if cur:
                out.append(cur)
            cur = []
        else:
            cur.append(d)
    if cur:
        out.append(cur)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--block", type=int, default=None, help="index of the flush-delimited block to use (default: "
                    "the last block of the most common length = one timed replay of the step)")
    ap.add_argument("--slack", type=float, default=1.5)
    ap.add_argument("--traffic-out", default=None,
                    help="write DRAM bytes per launch of the attention call sites (bench.py roofline 'traffic')")
    a = ap.parse_args()
    blocks = [b for b in steps(load(a.csv)) if len(b) > 20]
    if a.block is None:
        # the timed replays are flush-delimited single steps; earlier blocks
        # hold several back-to-back steps: the step is the shortest period of
        # the launch-name sequence, taken from the last block
        blk = blocks[-1]
        names = [d["name"] for d in blk]
        # smallest period (the capture may end mid-step: a truncated last repeat is allowed)
        per = next(p for p in range(1, len(names) + 1) if all(names[i] == names[i % p] for i in range(len(names))))
        k = len(names) // per
        step = blk[(k - 1) * per:k * per]
    else:
        step = blocks[a.block]
    rd = sum(d.get("dram__bytes_read.sum", 0.0) for d in step)
    wr = sum(d.get("dram__bytes_write.sum", 0.0) for d in step)
    us = sum(d.get("gpu__time_duration.sum", 0.0) for d in step) / 1e3
    sys.path.insert(0, ROOT)
    from paper_2110_10802_b200.bert import BertLayerConfig, fused_step_bytes

    sched = fused_step_bytes(BertLayerConfig(), B, S)
    mv = json.load(open(os.path.join(ROOT, "tests", "golden", "movement_volume.json")))
    ref = mv["bert_c2"]["fwd_bwd_library_bytes"] / 2
    print("| # | kernel | grid | DRAM read MB | DRAM write MB | us |\n|---|---|---|---|---|---|")
    for i, d in enumerate(step):
        nm = d["name"].split("(")[0].replace("void ", "").replace("dfx::<unnamed>::", "")[:60]
        print(f"| {i} | `{nm}` | {d['grid']} | {d.get('dram__bytes_read.sum', 0) / 1e6:.2f} | "
              f"{d.get('dram__bytes_write.sum', 0) / 1e6:.2f} | {d.get('gpu__time_duration.sum', 0) / 1e3:.1f} |")
    meas = rd + wr
    if a.traffic_out:
        def dram(d):
            return d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tr = {}
        for i, d in enumerate(step):
            if "attn_fwd" in d["name"]:
                tr["fwd.attention"] = tr.get("fwd.attention", 0.0) + dram(d)
            elif "attn_bwd" in d["name"]:
                tr["bwd.attention"] = tr.get("bwd.attention", 0.0) + dram(d)
                # the dQ GEMM over the stored dSᵀ follows the key-strip kernel in the same call
                if "kstrip" in d["name"] and i + 1 < len(step) and "tc_gemm_kernel<64" in step[i + 1]["name"]:
                    tr["bwd.attention"] += dram(step[i + 1])
        tr["source"] = "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (tools/reconcile_bytes.py)"
        json.dump(tr, open(a.traffic_out, "w"), indent=1)
    print(f"\n| quantity | bytes per step | vs schedule |\n|---|---|---|")
    print(f"| measured (ncu DRAM read + write, {len(step)} launches, {us:.1f} us serialised) | {meas / 1e6:.1f} MB | "
          f"{meas / sched:.3f} |")
    print(f"| schedule (BertEncoderLayer.step_bytes, compulsory) | {sched / 1e6:.1f} MB | 1.000 |")
    print(f"| reference unfused (dfir ir.movement_volume, bf16) | {ref / 1e6:.1f} MB | {ref / sched:.3f} |")
    print(f"| measured DRAM writes alone | {wr / 1e6:.1f} MB | (most writes stay in the 126 MB L2 within a step; "
          f"their write-back lands in the next L2 flush) |")
    print(f"\nmeasured / reference unfused = {meas / ref:.4f}")
    if meas > a.slack * sched:
        print(f"FAIL: measured traffic exceeds {a.slack}x the compulsory bytes", file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()
