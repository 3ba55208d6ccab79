"""Condense the compute-sanitizer logs of tools/sanitize.sh
(gpurun_out/sanitize_<tool>.log + .pytest) into a markdown summary:
per tool the error summary line, the pytest outcome, and the distinct
kernels named in any report.  Usage: python tools/sanitize_summary.py [dir]."""

import collections
import glob
import os
import re
import sys


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    print("| tool | sanitizer summary | pytest | kernels with reports |\n|---|---|---|---|")
    for log in sorted(glob.glob(os.path.join(d, "sanitize_*.log"))):
        tool = os.path.basename(log)[len("sanitize_"):-4]
        text = open(log, errors="replace").read()
        summ = re.findall(r"(?:ERROR|RACECHECK) SUMMARY: ([^\n]+)", text)
        kern = collections.Counter(re.findall(r"in (?:void )?([A-Za-z_:<>0-9, ]+?)\(", text))
        pt = os.path.join(d, f"sanitize_{tool}.pytest")
        outcome = ""
        if os.path.exists(pt):
            lines = [ln.strip() for ln in open(pt, errors="replace") if ln.strip()]
            outcome = next((ln for ln in reversed(lines) if "passed" in ln or "failed" in ln), lines[-1] if lines else "")
        ks = ", ".join(f"`{k.split('::')[-1]}` x{n}" for k, n in kern.most_common(6)) or "none"
        print(f"| {tool} | {'; '.join(summ) or 'no summary line'} | {outcome} | {ks} |")


if __name__ == "__main__":
    main()
