"""Generate the readahead-law fixtures under tests/golden/windows/ by running the
reference's own HostOs (host_os.py:106-152, the ondemand window law) on single read
streams.  Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_windows.py

Each fixture is one stream: a file size, the OS page (= the GPU page on our side), the
window cap and the list of reads (offset, size), with the reference's window_history and
SSD bytes after every read.  tests/test_readahead_law.py replays the same reads through
the oracle's restatement (CPU) and tests/test_gpu_readahead.py through the device (one TB
whose program is the read list), both with io.ra_clamp=eof (the reference's clamp).
The scenarios are the reference's own tests/test_host_os.py:51-141 and acceptance
criterion 1 (tests/test_acceptance.py:54-74), plus longer and unaligned streams.
"""

from __future__ import annotations

import json
import os
import random

from gpuiosim.devices import SsdModel
from gpuiosim.host_os import HostOs
from gpuiosim.metrics import Metrics
from gpuiosim.simcore import EventQueue

KiB, MiB = 1 << 10, 1 << 20
PAGE = 4096
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "windows")


def run_stream(file_bytes: int, ra_max: int, reads: list[tuple[int, int]]) -> dict:
    q = EventQueue()
    ssd = SsdModel(2_800_000_000, 80_000, 32)
    m = Metrics()
    host = HostOs(q, ssd, {0: file_bytes}, PAGE, 1 << 34, ra_max, 100, m)
    hist_after, ssd_after = [], []
    for off, size in reads:
        host.pread(0, off, size, q.now, lambda n, t, b: None)
        while (ev := q.pop()) is not None:  # each read completes before the next (one stream)
            ev.action(ev.fire_at)
        hist_after.append(len(m.window_history))
        ssd_after.append(ssd.bytes_read)
    return {"file_bytes": file_bytes, "page": PAGE, "ra_max": ra_max, "reads": reads,
            "window_history": list(m.window_history), "history_len_after_read": hist_after,
            "ssd_bytes_after_read": ssd_after}


def pages(first: int, count: int, size: int = PAGE) -> list[tuple[int, int]]:
    return [(p * PAGE, size) for p in range(first, first + count)]


def scenarios() -> dict:
    s = {}
    # acceptance criterion 1: 4 KiB reads of a 4 MiB file, cap 128 KiB (the criterion reads
    # pages 0..255; here also the whole file, to EOF)
    s["criterion1_256"] = (4 * MiB, 128 * KiB, pages(0, 256))
    s["criterion1_to_eof"] = (4 * MiB, 128 * KiB, pages(0, 1024))
    # tests/test_host_os.py
    s["cold_4k"] = (4 * MiB, 128 * KiB, pages(0, 1))
    s["marker_once"] = (4 * MiB, 128 * KiB, [(0, PAGE), (PAGE, PAGE), (PAGE, PAGE)])
    s["cached_rewind"] = (4 * MiB, 128 * KiB, pages(0, 64) + pages(0, 8) + pages(64, 1))
    s["nonsequential_reset"] = (16 * MiB, 128 * KiB, [(0, PAGE), (500 * PAGE, PAGE), (501 * PAGE, PAGE)])
    s["context_recovery"] = (16 * MiB, 128 * KiB, [(0, PAGE), (1000 * PAGE, PAGE), (PAGE, PAGE)])
    s["request_at_ra_max"] = (16 * MiB, 128 * KiB, [(0, 256 * KiB), (256 * KiB, 256 * KiB)])
    s["eof_clamp"] = (2 * PAGE, 128 * KiB, [(0, PAGE), (PAGE, PAGE)])
    # the bench's law: 64 KiB requests, windows up to 16 MiB, one 16 MiB stream
    s["req64k_cap16m"] = (16 * MiB, 16 * MiB, [(o, 64 * KiB) for o in range(0, 16 * MiB, 64 * KiB)])
    s["req64k_cap1m"] = (8 * MiB, 1 * MiB, [(o, 64 * KiB) for o in range(0, 8 * MiB, 64 * KiB)])
    s["req16k_cap256k"] = (2 * MiB + 12 * KiB, 256 * KiB,
                           [(o, 16 * KiB) for o in range(0, 2 * MiB + 12 * KiB, 16 * KiB)])
    # unaligned requests (pages shared by consecutive reads) and a short EOF tail
    s["unaligned_6k"] = (1 * MiB + 1000, 128 * KiB,
                         [(o, 6 * KiB) for o in range(0, 1 * MiB + 1000, 6 * KiB)])
    # two sequential runs separated by a jump, then a return to the first run's end
    s["two_runs"] = (8 * MiB, 64 * KiB, pages(0, 40) + pages(1000, 40) + pages(40, 20))
    # seeded random page reads (mostly non-sequential, some accidental continuations)
    rng = random.Random(7)
    rr, p = [], 0
    for _ in range(200):
        p = p + 1 if rng.random() < 0.5 else rng.randrange(0, 2048)
        rr.append((p * PAGE, PAGE))
    s["random_mix"] = (8 * MiB, 64 * KiB, rr)
    return s


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    for name, (fb, ra, reads) in scenarios().items():
        rec = run_stream(fb, ra, reads)
        rec["name"] = name
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump(rec, fh)
        print(f"{name}: {len(reads)} reads, windows {rec['window_history'][:8]}"
              f"{'...' if len(rec['window_history']) > 8 else ''}")


if __name__ == "__main__":
    main()
