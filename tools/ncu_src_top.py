"""Top SASS instructions by warp-stall samples from an ncu source-page CSV
(``ncu -i rep --page source --csv --print-source sass``)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    for a, b in zip(starts, starts[1:]):
        print("=====", rows[a][1][:100])
        section(rows[a:b], top)


def section(rows, top):
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0] != "Address"]
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    print(f"{len(data)} instructions, {tot} stall samples")
    data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:top]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        print(f"{100 * s / max(tot, 1):5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:70]:70s} "
              f"exec={r[ix['Instructions Executed']]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
