"""Top SASS instructions by warp-stall samples from an ncu source-page CSV:
python tools/ncu_src_top.py src.csv [N]"""
import csv
import sys

REASONS = ['stall_long_sb', 'stall_short_sb', 'stall_wait', 'stall_barrier', 'stall_selected', 'stall_not_selected',
           'stall_math', 'stall_mio', 'stall_branch_resolving', 'stall_lg', 'stall_membar', 'stall_sleeping',
           'stall_dispatch', 'stall_drain', 'stall_no_inst', 'stall_tex', 'stall_misc']


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    data, seen = [], set()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r[0] == "Address":
            continue
        if r[0] in seen:
            break
        seen.add(r[0])
        data.append(r)
    col = 'Warp Stall Sampling (All Samples)'
    total = sum(int(r[ix[col]] or 0) for r in data)
    top = sorted(data, key=lambda r: -int(r[ix[col]] or 0))[:n]
    print(f"{len(data)} instructions, {total} samples")
    for r in top:
        s = int(r[ix[col]] or 0)
        rs = {k[6:]: int(r[ix[k]] or 0) for k in REASONS if k in ix and int(r[ix[k]] or 0) >= max(2, s // 10)}
        print(f"{r[0][-5:]} {s:5d} ({100 * s / total:4.1f}%) {r[ix['Source']][:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
