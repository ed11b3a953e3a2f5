"""CLI and harness host logic (no GPU): argument handling, config errors -> exit 2."""

import pytest

from paper_2109_05366_b200 import cli
from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.experiments import PRESETS, run_preset
from paper_2109_05366_b200.errors import GfsError


def test_bad_key_exits_2(capsys):
    assert cli.main(["run", "--set", "no.such=1"]) == 2
    assert "unknown config key" in capsys.readouterr().err


def test_unknown_preset_is_an_error(tmp_path):
    with pytest.raises(GfsError):
        run_preset("fig99", ExperimentConfig(), str(tmp_path))


def test_preset_arms_match_the_reference_shapes():
    base = ExperimentConfig()
    labels = [l for l, _c in PRESETS["fig8"](base)]
    assert labels == [f"prefetch-{k * 1024}" for k in (0, 12, 28, 60, 124, 252)]
    arms = dict(PRESETS["fig10micro"](base))
    assert arms["lra-prefetch"]["gpufs.policy"] == "per-tb-lra"
    assert arms["baseline-4k"]["gpufs.prefetch_bytes"] == 0
    assert arms["global-prefetch"]["gpufs.cache_bytes"] == 98_304_000 // 2
    bench = list(PRESETS["bench"](base.copy_with({"workload.scale": 0.01})))
    assert len(bench) == 14 * 3


def _write_trace(path, recs):
    with open(path, "w") as fh:
        fh.write("# tb_id file_id offset size\n")
        for r in recs:
            fh.write(" ".join(map(str, r)) + "\n")


def test_replay_reads_every_traced_byte_on_host(tmp_path):
    """`replay` (the reference's `gpuiosim replay`, cli.py:81-87): host threads pread every
    trace record, no GPU in the loop; user bytes = sum of record sizes, one pread each."""
    from paper_2109_05366_b200.runtime import Simulation
    fb = 1 << 20
    recs = [(tb, f, k * 65536 + tb * 4096, 65536 if k < 7 else 20000)
            for tb in range(6) for f in range(2) for k in range(8) if k * 65536 + tb * 4096 + 65536 <= fb]
    trace = str(tmp_path / "t.txt")
    _write_trace(trace, recs)
    cfg = ExperimentConfig({"mode.replay_trace": trace, "workload.file_bytes": fb,
                            "workload.n_files": 2, "io.dir": str(tmp_path), "rpc.n_workers": 4})
    sim = Simulation(cfg, 42)
    rep = sim.run()
    assert rep["user_bytes"] == sum(r[3] for r in recs)
    assert rep["ssd_requests"] == len(recs) and rep["greads"] == 0
    assert rep["io_bandwidth_bps"] > 0


def test_replay_cli_and_trace_errors(tmp_path, capsys):
    fb = 1 << 20
    trace = str(tmp_path / "t.txt")
    _write_trace(trace, [(0, 0, 0, 4096), (1, 0, 4096, 8192)])
    out = str(tmp_path / "r.csv")
    assert cli.main(["replay", trace, "--set", f"workload.file_bytes={fb}", "--set",
                     f"io.dir={tmp_path}", "--set", "repetitions=1", "--out", out]) == 0
    assert open(out).read().count("\n") == 3  # header, one rep, the mean row
    bad = str(tmp_path / "bad.txt")
    _write_trace(bad, [(0, 3, 0, 4096)])  # file 3 does not exist (trace_workload)
    assert cli.main(["replay", bad, "--set", f"workload.file_bytes={fb}", "--set",
                     f"io.dir={tmp_path}"]) == 2
    assert "unknown file" in capsys.readouterr().err
    _write_trace(bad, [(0, 0, fb - 4096, 8192)])  # past EOF
    assert cli.main(["replay", bad, "--set", f"workload.file_bytes={fb}", "--set",
                     f"io.dir={tmp_path}"]) == 2


def test_mosaic_and_fig3_presets_exist():
    base = ExperimentConfig()
    arms = dict(PRESETS["mosaic"](base))
    assert set(arms) == {"random-page-4096", "random-page-65536"}
    assert all(c["workload.kind"] == "random" and c["gpufs.prefetch_bytes"] == 0 for c in arms.values())
    assert "fig3" in PRESETS
