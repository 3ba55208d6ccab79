"""Warp-stall samples of an ncu source-page CSV (SASS) grouped into segments
delimited by barrier / mbarrier / TMEM-load instructions, with the dominant
stall reasons per segment: python tools/ncu_segments.py src.csv"""
import csv
import sys

REASONS = ['stall_long_sb', 'stall_short_sb', 'stall_wait', 'stall_barrier', 'stall_selected', 'stall_not_selected',
           'stall_math', 'stall_mio', 'stall_branch_resolving', 'stall_lg']


def main(path):
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
    total = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data)
    print(f"{len(data)} instructions, {total} samples")
    seg, segtot, start = {k: 0 for k in REASONS}, 0, data[0][0][-5:]
    for r in data:
        src = r[ix['Source']]
        segtot += int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
        for k in REASONS:
            seg[k] += int(r[ix[k]] or 0)
        if any(t in src for t in ['BAR.SYNC', 'TRYWAIT', 'LDTM', 'SYNCS.ARRIVE']):
            end = r[0][-5:] + ' ' + (src.split()[1] if src.startswith('@') else src.split()[0])
            if segtot > 15:
                print(f"{start:>24s} .. {end:24s} {segtot:5d} ({100 * segtot / total:4.1f}%) " +
                      ' '.join(f"{k[6:]}:{v}" for k, v in seg.items() if v >= 4))
            seg, segtot, start = {k: 0 for k in REASONS}, 0, end


if __name__ == "__main__":
    main(sys.argv[1])
