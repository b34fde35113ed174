"""Instruction mix and warp-stall reasons of one kernel from an ncu source-page CSV
(`ncu -i rep --page source --csv --print-source sass`), as kept under profiles/.

  python tools/ncu_source_summary.py <src.csv[.gz]> <kernel-substring> <out.json>
"""
from __future__ import annotations

import collections
import csv
import gzip
import io
import json
import sys


def main():
    path, pat, out = sys.argv[1:4]
    raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    kern, cur = [], None
    for r in csv.reader(raw):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            kern.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    k = next(k for k in kern if pat in k["name"])
    h = k["hdr"]
    S, I, W = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    mix, samp, stall = collections.Counter(), collections.Counter(), collections.Counter()
    for r in k["rows"]:
        op = r[S].strip().split()
        if not op:
            continue
        base = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        mix[base] += int(r[I] or 0)
        samp[base] += int(r[W] or 0)
        for i in cols:
            stall[h[i][6:]] += int(r[i] or 0)
    ti, ts, tst = sum(mix.values()), sum(samp.values()), sum(stall.values())
    res = {"kernel": k["name"], "instructions_executed": ti,
           "mix_pct": {o: round(100 * n / ti, 2) for o, n in mix.most_common(20)},
           "stall_samples_pct_by_opcode": {o: round(100 * n / ts, 2) for o, n in samp.most_common(12)},
           "stall_reasons_pct": {c: round(100 * n / tst, 2) for c, n in stall.most_common(12)}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res)[:600])


if __name__ == "__main__":
    main()
