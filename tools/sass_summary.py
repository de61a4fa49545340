"""Summarise ncu source-page SASS CSVs (tools/prof_small.sh) into markdown:
warp-instruction totals, stall-reason shares and the opcode mix.

    python tools/sass_summary.py gpurun_out/small/dual_sass.csv.gz [...] > profiles/rNN_transform_sass.md
"""
import collections
import csv
import gzip
import re
import sys


def summarise(path):
    lines = gzip.open(path, "rt").read().splitlines()
    rows = list(csv.reader(lines[1:]))
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (KeyError, ValueError):
            return 0.0
    tot = sum(f(r, "Instructions Executed") for r in rows)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {s: sum(f(r, s) for r in rows) for s in stalls}
    st = sum(agg.values()) or 1.0
    ops = collections.Counter()
    for r in rows:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ix["Source"]].strip())
        if m:
            ops[m.group(2)] += f(r, "Instructions Executed")
    out = [f"### {path.split('/')[-1]}", "", f"warp instructions executed: {tot / 1e6:.2f} M", "",
           "| stall reason | share of samples |", "|---|---|"]
    out += [f"| {k[6:]} | {100 * v / st:.1f} % |" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]]
    out += ["", "| opcode | share of instructions |", "|---|---|"]
    out += [f"| {k} | {100 * v / tot:.1f} % |" for k, v in ops.most_common(16)]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print("\n".join(summarise(p) for p in sys.argv[1:]))
