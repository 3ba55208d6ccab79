"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
of ``bench.py`` into the per-kernel table kept under profiles/.

The bench captures one training step into a CUDA graph; the last
``--per-step`` launches of the list are the final replayed step (the L2
flush kernel, torch's fill, is excluded).  Launches are printed in order with
their share of the step; ncu times are cold-cache and serialised, so shares
(not absolutes) are what to compare with bench.py's event timings."""

import argparse
import csv


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append(d)
    return data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--per-step", type=int, default=0, help="launches per step (0: after the last flush)")
    a = ap.parse_args()
    data = load(a.csv)
    # last step = launches after the last torch fill (the L2 flush)
    idx = [i for i, d in enumerate(data) if "FillFunctor" in d["Kernel Name"]]
    step = data[idx[-1] + 1:] if idx and not a.per_step else data[-a.per_step:]
    if not a.per_step:  # several back-to-back replays after the flush: keep the last period
        names = [d["Kernel Name"] for d in step]
        per = next(p for p in range(1, len(names) + 1) if all(names[i] == names[i % p] for i in range(len(names))))
        k = len(names) // per
        step = step[(k - 1) * per:k * per]
    tot = sum(float(d["Metric Value"]) for d in step)
    print(f"| # | kernel | grid | block | us | share |\n|---|---|---|---|---|---|")
    for i, d in enumerate(step):
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dfx::<unnamed>::", "")
        us = float(d["Metric Value"]) / 1e3
        print(f"| {i} | `{name}` | {d['Grid Size']} | {d['Block Size']} | {us:.1f} | {us * 1e3 / tot:.1%} |")
    print(f"\nstep total (serialised, cold L2): {tot / 1e3:.1f} us over {len(step)} launches")


if __name__ == "__main__":
    main()
