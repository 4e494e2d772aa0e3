"""Dataset generator / TSV writer and the CLI's argument handling (no GPU needed)."""
import os
import subprocess

import numpy as np
import pytest

import paper_1809_07858_b200 as pf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1809_07858_b200", "shouji-b200")


def run(*args, stdin=None):
    r = subprocess.run([CLI, *args], input=stdin, capture_output=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


@pytest.mark.parametrize("seed,count,m,lo,hi", [(1809078580, 20000, 100, 0, 10), (5, 3000, 37, 3, 3),
                                                (9, 2000, 250, 0, 50), (2, 500, 1, 0, 1)])
def test_generate_pairs_matches_restated_reference(oracle, seed, count, m, lo, hi):
    # generate_pairs (dataset.cpp:71-126); the oracle's restatement is pinned to the
    # reference library by tests/test_oracle.py
    ds = pf.generate_pairs(seed, count, m, lo, hi)
    t, p = oracle.generate_pairs(seed, count, m, lo, hi)
    assert (ds.text() == t).all() and (ds.pattern() == p).all()
    assert ds.source == f"gen(seed={seed},count={count},len={m},edits={lo}..{hi})"


def test_generate_pairs_parameter_errors():
    for args in [(1, 0, 10, 0, 1), (1, 5, 0, 0, 1), (1, 5, 10, 3, 2), (1, 5, 10, 0, 11)]:
        with pytest.raises(pf.invalid_parameters_error):
            pf.generate_pairs(*args)


def test_cli_gen_writes_reference_tsv(oracle, tmp_path):
    rc, out, _ = run("gen", "--seed", "7", "--count", "300", "--len", "50", "--edits", "0..6")
    assert rc == 0
    t, p = oracle.generate_pairs(7, 300, 50, 0, 6)
    expect = b"".join(t[i].tobytes() + b"\t" + p[i].tobytes() + b"\n" for i in range(300))
    assert out == expect
    f = tmp_path / "pairs.tsv"
    rc, _, _ = run("gen", "--seed", "7", "--count", "300", "--len", "50", "--edits", "0..6",
                   "--pairs", str(f))
    assert rc == 0 and f.read_bytes() == expect


@pytest.mark.parametrize("args", [
    [], ["bogus"], ["filter", "--count", "5", "--len", "10"],                       # no threshold
    ["filter", "--count", "5", "--len", "10", "--e", "1", "--e-percent", "5"],     # both
    ["filter", "--count", "5", "--len", "10", "--e", "1", "--width", "9"],         # range
    ["filter", "--e", "1"],                                                        # no input
    ["gen", "--count", "5", "--len", "10"],                                        # no --edits
    ["gen", "--count", "5", "--len", "10", "--edits", "4..2"],                     # inverted
    ["bench", "--len", "100"],                                                     # no --e
])
def test_cli_usage_errors_exit_1(args):
    rc, _, err = run(*args)
    assert rc == 1 and b"usage error" in err


def test_cli_data_error_exit_2(tmp_path):
    rc, _, err = run("gen", "--seed", "1", "--count", "5", "--len", "10", "--edits", "0..11")
    assert rc == 1  # cannot plant more edits than bases: invalid parameters
    rc, _, err = run("filter", "--pairs", str(tmp_path / "missing.tsv"), "--e", "1")
    assert rc == 2 and b"error" in err
