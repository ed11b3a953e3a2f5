"""The product never routes through the checker: no module of the package (or the native
sources) imports, loads or links anything under oracle/."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2109_05366_b200")


def test_package_does_not_reference_the_oracle():
    offenders = []
    for dirpath, _dirs, files in os.walk(PKG):
        for f in files:
            if not f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                continue
            text = open(os.path.join(dirpath, f), errors="replace").read()
            if re.search(r"\boracle\b|gfs_oracle|orc_", text):
                offenders.append(os.path.relpath(os.path.join(dirpath, f), ROOT))
    assert not offenders, offenders


def test_build_links_no_oracle_object():
    from paper_2109_05366_b200 import build
    assert all("oracle" not in s for s in build.SOURCES)
