"""Summarise an ncu --set full capture of gread_driver into profiles/<round>/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01 --user-bytes N --tag NAME
"""

import argparse
import csv
import io
import json
import os
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
        "smsp__average_warp_latency_issue_stalled_barrier.ratio",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_membar"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("outdir")
    ap.add_argument("--user-bytes", type=int, required=True)
    ap.add_argument("--tag", default="gread")
    ap.add_argument("--workload", default="")
    ap.add_argument("--source-top", type=int, default=25)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    def num(v):
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return v

    d = {h: (num(v), u) for h, u, v in zip(hdr, units, vals)}
    out = {k: {"value": d[k][0], "unit": d[k][1]} for k in KEYS if k in d}
    dur_ms = out["gpu__time_duration.sum"]["value"] * SCALE[out["gpu__time_duration.sum"]["unit"]]
    rd = out["dram__bytes_read.sum"]["value"] * SCALE[out["dram__bytes_read.sum"]["unit"]]
    wr = out["dram__bytes_write.sum"]["value"] * SCALE[out["dram__bytes_write.sum"]["unit"]]
    summary = {
        "kernel": "gread_driver<256>", "workload": a.workload,
        "capture": "ncu --replay-mode application --set full --import-source on --clock-control none "
                   "-k regex:gread_driver -c 1",
        "duration_ms": dur_ms, "user_bytes": a.user_bytes,
        "user_GBps_in_profiled_pass": a.user_bytes / (dur_ms / 1e3) / 1e9,
        "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
        "dram_bytes_per_user_byte": (rd + wr) / a.user_bytes,
        "metrics": out,
    }
    os.makedirs(a.outdir, exist_ok=True)
    with open(os.path.join(a.outdir, f"ncu_{a.tag}_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    # stall stack by reason and the hottest source lines (warp-state samples)
    summary["stall_samples"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(num(v))
                                for k, v in zip(hdr, vals)
                                if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                                and not k.endswith("_not_issued") and num(v) not in ("", 0, 0.0)}
    src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hot = []
    # the page lists one section per source file ("File Path" / "File Name" rows), each with
    # its own header row
    cur, iS = "?", None
    for r in srows:
        if r and r[0] in ("File Path", "File Name") and len(r) > 1:
            cur = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            iS = r.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in r else None
            continue
        if iS is not None and len(r) > iS and r[0] not in ("", "-") and r[2] == "-":
            try:
                hot.append((int(r[iS]), f"{cur}:{int(r[0])}", r[1].strip()[:100]))
            except ValueError:
                pass
    if hot:
        tot = sum(h[0] for h in hot) or 1
        hot.sort(reverse=True)
        summary["hot_source_lines"] = [{"line": ln, "samples": n, "share": round(n / tot, 4), "source": sl}
                                       for n, ln, sl in hot[:a.source_top]]
    with open(os.path.join(a.outdir, f"ncu_{a.tag}_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    det = subprocess.run(["ncu", "-i", a.rep, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    with open(os.path.join(a.outdir, f"ncu_{a.tag}_details.csv"), "w") as fh:
        fh.write(det)
    print(json.dumps({k: v for k, v in summary.items() if k != "metrics"}, indent=1))


if __name__ == "__main__":
    main()
