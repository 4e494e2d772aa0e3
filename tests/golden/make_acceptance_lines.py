#!/usr/bin/env python
"""Expected output lines of the reference's acceptance criteria 1-5 and 7
(proj/tests/acceptance_tests.cpp, unmodified), produced by the unmodified
reference library: integration/_build/acceptance_ref (integration/Makefile).
Timing fragments are normalised away (see normalise()); the committed file is
tests/golden/acceptance_ref_lines.txt, which tests/test_gpu_reference_suites.py
compares against integration/_build/acceptance_b200 (the same source linked
against the B200 drop-in) on the GPU box.

python tests/golden/make_acceptance_lines.py
"""
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "acceptance_ref_lines.txt")
CRITERIA = [1, 2, 3, 4, 5, 7]


def normalise(line: str) -> str:
    """Drop wall-clock fragments: the trailing "; <t> s" of criteria 2/5, criterion 1's
    "golden pair e=3, <t> ms" duration and its "runs in milliseconds" verdict (the B200
    build's first call also creates the CUDA context, ~1 s once per process)."""
    line = re.sub(r"; [0-9.]+ s$", "", line.rstrip())
    line = re.sub(r"golden pair e=3, [0-9.]+ ms", "golden pair e=3", line)
    line = line.replace("failed: runs in milliseconds; ", "")
    return line


def run(binary, criterion):
    r = subprocess.run([binary, str(criterion)], capture_output=True, text=True, timeout=1800)
    lines = [normalise(x) for x in r.stdout.splitlines() if x.startswith(("PASS", "FAIL"))]
    assert len(lines) == 1, r.stdout + r.stderr
    return lines[0]


def main():
    binary = os.path.join(ROOT, "integration", "_build", "acceptance_ref")
    if not os.path.exists(binary):
        sys.exit("build integration/ first (make -C integration)")
    with open(OUT, "w") as f:
        for c in CRITERIA:
            f.write(run(binary, c) + "\n")
    print(open(OUT).read())


if __name__ == "__main__":
    main()
