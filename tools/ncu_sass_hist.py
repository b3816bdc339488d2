"""Opcode histogram (executed warp instructions) and top stall sites of an ncu report.

  python tools/ncu_sass_hist.py report.ncu-rep [kernel-index]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    h = rows[hi]
    ii, si, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    seen, data = set(), []
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[0] in seen:
            continue
        seen.add(r[0])
        data.append(r)
    c = collections.Counter()
    for r in data:
        op = r[src].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += f(r[ii])
    tot = sum(c.values())
    print("total warp-inst", tot)
    for k, v in c.most_common(25):
        print(f"{k:12s} {v:12.0f} {100 * v / tot:5.1f}%")
    print("--- top stall sites")
    for r in sorted(data, key=lambda r: -f(r[si]))[:25]:
        print(f"{r[si]:>6s} {r[ii]:>9s}  {r[src][:90]}")


if __name__ == "__main__":
    main()
