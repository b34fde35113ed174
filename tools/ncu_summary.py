"""Summarise ncu captures into the JSON files kept under profiles/.

  python tools/ncu_summary.py full  <report.ncu-rep> <out.json> "<capture command>"
  python tools/ncu_summary.py launches <launches.csv> <out.json> "<capture command>"

`full` keeps, per captured kernel, the time, DRAM bytes, tensor-pipe / issue
utilisation, L2 <-> SM traffic and the top warp-stall reasons; `launches`
groups a `--metrics gpu__time_duration.sum` launch list by kernel name (count,
total and mean time, share of the listed time).
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_op_read_hit_rate.pct", "derived__lts__lts2xbar_bytes.sum.per_second",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x",
]


def full(rep, out, cmd):
    # a .ncu-rep, or the `--page raw --csv` export of one (made on the GPU box when the
    # report itself is too large to bring back)
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        d = dict(zip(head, v))
        u = dict(zip(head, units))
        k = OrderedDict(kernel=d.get("Kernel Name", "")[:160])
        for m in FULL_METRICS:
            if m in d:
                k[m] = f"{d[m]} {u.get(m, '')}".strip()
        st = []
        for name in head:
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
                try:
                    st.append((name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                               float(d[name])))
                except ValueError:
                    pass
        st.sort(key=lambda x: -x[1])
        k["top_stalls_per_issue"] = OrderedDict((a, round(b, 3)) for a, b in st[:6])
        kernels.append(k)
    json.dump({"capture": cmd, "report": rep.split("/")[-1], "kernels": kernels}, open(out, "w"), indent=1)


def launches(path, out, cmd):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = OrderedDict()
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:120]
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = val * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        a = agg.setdefault(name, {"launches": 0, "total_ms": 0.0})
        a["launches"] += 1
        a["total_ms"] += ms
        total += ms
    for a in agg.values():
        a["mean_ms"] = a["total_ms"] / a["launches"]
        a["share"] = a["total_ms"] / total if total else None
    ordered = OrderedDict(sorted(agg.items(), key=lambda kv: -kv[1]["total_ms"]))
    json.dump({"capture": cmd, "note": "cold-cache, serialised per-launch times (ncu); shares, not absolutes, "
                                       "compare with bench.py", "total_ms": total, "kernels": ordered},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    mode, src, dst, cmd = sys.argv[1:5]
    (full if mode == "full" else launches)(src, dst, cmd)
