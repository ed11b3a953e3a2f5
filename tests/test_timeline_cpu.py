"""Timeline analysis (host logic, no GPU): interval unions and the overlap measures."""

import numpy as np

from paper_2109_05366_b200 import timeline


def rec(kind, cta, tb, nbytes, t0, t1):
    return [(kind << 56) | (cta << 32) | tb, nbytes, t0, t1]


def test_decode_round_trip():
    r = np.array([rec(2, 591, 1023, 65536, 10, 20)], dtype=np.int64)
    d = timeline.decode(r)
    assert (d["kind"][0], d["cta"][0], d["tb"][0], d["bytes"][0]) == (2, 591, 1023, 65536)


def test_overlap_measures():
    # transfers outstanding over [0, 100) and [200, 300); compute over [50, 150) and [250, 260)
    r = np.array([rec(0, 0, 0, 4096, 0, 60), rec(0, 1, 1, 4096, 40, 100), rec(0, 0, 0, 4096, 200, 300),
                  rec(2, 2, 2, 4096, 50, 150), rec(2, 3, 3, 4096, 250, 260)], dtype=np.int64)
    s = timeline.summary(r)
    assert s["span_ns"] == 300 and s["ctas"] == 4 and s["rpcs"] == 3
    assert s["io_busy_frac"] == round(200 / 300, 4)
    assert s["consume_overlap_frac"] == round((50 + 10) / 110, 4)  # [50,100) and [250,260)
    assert s["cta_consume_frac"] == round(110 / (300 * 4), 4)


def test_chrome_trace(tmp_path):
    import json
    r = np.array([rec(0, 0, 0, 1, 1000, 3000), rec(1, 0, 0, 1, 0, 4000)], dtype=np.int64)
    p = tmp_path / "t.json"
    timeline.chrome_trace(r, str(p))
    ev = json.load(open(p))["traceEvents"]
    assert [e["name"] for e in ev] == ["rpc", "gread"] and ev[0]["ts"] == 1.0 and ev[1]["dur"] == 4.0
