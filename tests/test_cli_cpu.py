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
