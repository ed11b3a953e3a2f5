"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file X`):
launches and total / mean device time per kernel, and each kernel's share.  Per-launch times
under ncu are cold-cache and serialised; only the shares are meant to be compared with the
live bench.

    python tools/launch_summary.py gpurun_out/launches_full.csv profiles/r01/ncu_launches_bench_full_summary.json
"""

import csv
import json
import sys
from collections import OrderedDict


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(src)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv, iu, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}
    per = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        ms = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        e = per.setdefault(name, {"launches": 0, "total_ms": 0.0})
        e["launches"] += 1
        e["total_ms"] += ms
    tot = sum(e["total_ms"] for e in per.values()) or 1.0
    for e in per.values():
        e["mean_ms"] = round(e["total_ms"] / e["launches"], 3)
        e["share"] = round(e["total_ms"] / tot, 4)
        e["total_ms"] = round(e["total_ms"], 3)
    summary = {"source": src, "launches": sum(e["launches"] for e in per.values()),
               "total_ms": round(tot, 3), "kernels": per}
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
