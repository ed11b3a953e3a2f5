"""Device timeline of a gread pass (mode.timeline): what every resident CTA was doing and
when, on the GPU's global timer — the evidence nsys would give for "PCIe transfer overlaps
compute" (nsys is not available on these boxes).

Records (include/gfs.h GFS_LOG_TIMELINE): (kind << 56 | cta << 32 | tb, bytes, t0, t1)
  rpc      a request published on the ring .. its data ready in HBM (transfer outstanding)
  gread    one gread call (page walk + waits + copies)
  consume  the fused consumer over the request's bytes
"""

from __future__ import annotations

import json

import numpy as np

KINDS = {0: "rpc", 1: "gread", 2: "consume"}


def decode(rec: np.ndarray) -> dict:
    rec = np.asarray(rec, dtype=np.int64).reshape(-1, 4)
    head = rec[:, 0]
    return {"kind": (head >> 56) & 0xFF, "cta": (head >> 32) & 0xFFFFFF, "tb": head & 0xFFFFFFFF,
            "bytes": rec[:, 1], "t0": rec[:, 2], "t1": rec[:, 3]}


def _union(t0: np.ndarray, t1: np.ndarray) -> list[tuple[int, int]]:
    """Disjoint sorted cover of the intervals [t0, t1)."""
    out: list[tuple[int, int]] = []
    for a, b in sorted(zip(t0.tolist(), t1.tolist())):
        if b <= a:
            continue
        if out and a <= out[-1][1]:
            if b > out[-1][1]:
                out[-1] = (out[-1][0], b)
        else:
            out.append((a, b))
    return out


def _length(iv: list[tuple[int, int]]) -> int:
    return sum(b - a for a, b in iv)


def _intersect(x: list[tuple[int, int]], y: list[tuple[int, int]]) -> int:
    i = j = tot = 0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if b > a:
            tot += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return tot


def summary(rec: np.ndarray) -> dict:
    """Overlap of transfers with compute.  `io_busy_frac`: share of the pass during which at
    least one transfer is outstanding; `consume_overlap_frac`: share of the time any CTA
    computes during which a transfer is outstanding too (1.0 = compute fully hidden under
    I/O); `cta_consume_frac`: CTA-time spent computing over CTA-time in the pass."""
    d = decode(rec)
    if len(d["t0"]) == 0:
        return {"records": 0}
    t_lo, t_hi = int(d["t0"].min()), int(d["t1"].max())
    span = max(1, t_hi - t_lo)
    out = {"records": int(len(d["t0"])), "span_ns": span,
           "ctas": int(len(np.unique(d["cta"])))}
    rpc = d["kind"] == 0
    con = d["kind"] == 2
    rpc_u = _union(d["t0"][rpc], d["t1"][rpc])
    out["rpcs"] = int(rpc.sum())
    out["io_busy_frac"] = round(_length(rpc_u) / span, 4)
    if rpc.any():
        lat = (d["t1"][rpc] - d["t0"][rpc]).astype(np.float64)
        out["rpc_latency_us"] = {"p50": round(float(np.percentile(lat, 50)) / 1e3, 2),
                                 "p99": round(float(np.percentile(lat, 99)) / 1e3, 2)}
        out["rpc_bytes_mean"] = int(d["bytes"][rpc].mean())
    if con.any():
        con_u = _union(d["t0"][con], d["t1"][con])
        out["consumes"] = int(con.sum())
        out["consume_busy_frac"] = round(_length(con_u) / span, 4)
        out["consume_overlap_frac"] = round(_intersect(con_u, rpc_u) / max(1, _length(con_u)), 4)
        out["cta_consume_frac"] = round(float((d["t1"][con] - d["t0"][con]).sum())
                                        / (span * out["ctas"]), 4)
    return out


def chrome_trace(rec: np.ndarray, path: str, max_events: int = 200_000) -> None:
    """Write a chrome://tracing / Perfetto JSON: one track per CTA."""
    d = decode(rec)
    t_lo = int(d["t0"].min()) if len(d["t0"]) else 0
    ev = []
    for i in range(min(len(d["t0"]), max_events)):
        ev.append({"name": KINDS.get(int(d["kind"][i]), "?"), "ph": "X", "pid": 0,
                   "tid": int(d["cta"][i]), "ts": (int(d["t0"][i]) - t_lo) / 1e3,
                   "dur": max(0, int(d["t1"][i]) - int(d["t0"][i])) / 1e3,
                   "args": {"tb": int(d["tb"][i]), "bytes": int(d["bytes"][i])}})
    with open(path, "w") as fh:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ms"}, fh)
