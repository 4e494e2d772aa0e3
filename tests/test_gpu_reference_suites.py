"""The reference's OWN tests, unmodified, run against the B200 build through its
C++ interface (integration/: the reference library with shouji_filter,
evaluate and run_bench swapped for integration/prefilter_b200.cpp, which calls
libshouji_b200.so):

* the unit suite (proj/tests/test_*.cpp except test_cli.cpp: 80 cases,
  175,923 checks) — the same count the unmodified reference passes
  (tests/test_oracle.py runs it on oracle/_ref);
* acceptance criteria 1-5 and 7 (proj/tests/acceptance_tests.cpp): every
  criterion line, timings aside, identical to the unmodified reference's
  (tests/golden/acceptance_ref_lines.txt, made by make_acceptance_lines.py from
  integration/_build/acceptance_ref). Criteria 2 and 5 call shouji_filter once
  per similar pair (~330k and ~1M calls): the drop-in's per-pair latency path.
Criterion 6 times CPU scaling with m and E and criterion 8 needs the reference
CLI (CLI11, absent); neither is a parity statement about this path.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(ROOT, "integration", "_build")
sys.path.insert(0, os.path.join(HERE, "golden"))

import make_acceptance_lines as mal  # noqa: E402


def _binary(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build with `make -C integration` (needs the reference tree)")
    return path


def test_reference_unit_suite_passes_on_b200():
    r = subprocess.run([_binary("unit_b200")], capture_output=True, text=True, timeout=900)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    m = re.search(r"cases (\d+) checks (\d+) failures (\d+)", tail)
    assert m and (int(m.group(1)), int(m.group(2)), int(m.group(3))) == (80, 175923, 0), tail


@pytest.mark.parametrize("criterion", mal.CRITERIA)
def test_reference_acceptance_criterion_lines_match(criterion):
    expected = open(os.path.join(HERE, "golden", "acceptance_ref_lines.txt")).read().splitlines()
    want = [x for x in expected if x.split(" (")[0].endswith(f"criterion {criterion}")]
    assert len(want) == 1
    assert mal.run(_binary("acceptance_b200"), criterion) == want[0]
