"""GPU: TSV ingest (load_pairs semantics), the exact oracle kernel and the CLI."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1809_07858_b200", "shouji-b200")

GOOD = b"ACGTACGT\tACGAACGT\nGGGGTTTT\tGGGGTTTA\nNNNNACGT\tACGTNNNN\n"

MALFORMED = [
    b"",                                        # no pairs in input
    b"\n",                                      # empty line: no tab
    b"ACGT ACGT\n",                             # no tab
    b"ACGT\tACGT\tACGT\n",                      # extra field
    b"\tACGT\n",                                # empty text
    b"ACGT\t\n",                                # empty pattern
    b"ACGT\tACGX\n",                            # illegal pattern byte
    b"acgt\tACGT\n",                            # lower case
    b"ACGT\tACG\n",                             # text/pattern length mismatch
    b"ACGT\tACGT\nACGTA\tACGTA\n",              # dataset length mismatch at line 2
    b"ACGT\tACGT\r\nACGT\tACGT\r\n",            # CRLF: '\r' is an illegal byte of the pattern
    GOOD + b"ACGTACGT\tACGTACGZ\n" + b"ACGT\n",  # illegal byte before a structural error
    GOOD + b"ACGT\n" + b"ACGTACGT\tACGTACGZ\n",  # structural error first
    GOOD + b"ACGTAC\tACGZ\n",                   # same line: pattern byte before lengths
    GOOD + b"ACGTACGX\tACG\n",                  # same line: text byte before lengths
    GOOD + b"ACGXACGT\t\n",                     # same line: text byte before empty pattern
    GOOD + b"\tACGXACGT\n",                     # same line: empty text first
    GOOD * 300 + b"ACGTACGT\tACGTACGT\tA\n",    # field count error deep in a file
    GOOD * 300 + b"ACGTACGT\tACGTANGU\n",       # illegal byte deep in a file
]


@pytest.mark.parametrize("i", range(len(MALFORMED)))
def test_load_pairs_errors_match_reference(gpu, reference, i):
    data = MALFORMED[i]
    st, _, _, msg = reference.load_pairs(data)
    assert st != 0
    with pytest.raises(gpu.error) as ei:
        gpu.load_pairs(data)
    assert str(ei.value) == msg, (data[:60], str(ei.value), msg)
    kind = {6: gpu.parse_error, 3: gpu.length_mismatch_error}[st]
    assert isinstance(ei.value, kind)


def test_load_pairs_good_input(gpu, reference):
    data = GOOD * 1000
    st, n, m, _ = reference.load_pairs(data)
    ds = gpu.load_pairs(data)
    assert st == 0 and len(ds) == n == 3000 and ds.length == m == 8
    lines = data.split(b"\n")[:-1]
    t = np.array([np.frombuffer(l.split(b"\t")[0], np.uint8) for l in lines])
    assert (ds.text() == t).all()


def test_banded_edit_distance_matches_reference(gpu, reference, oracle):
    rng = np.random.default_rng(4400)
    for m, e, rate in [(100, 5, 0.05), (100, 10, 0.2), (64, 64, 0.3), (65, 7, 0.1), (150, 15, 0.1),
                       (250, 25, 0.08), (1, 0, 0.5), (300, 40, 0.1), (37, 3, 0.0)]:
        n = 2000
        t = np.frombuffer(b"ACGTN", np.uint8)[rng.integers(0, 5, size=(n, m))]
        p = t.copy()
        for i in range(n):
            for _ in range(int(rng.integers(0, max(1, int(rate * m)) + 1))):
                pos = int(rng.integers(0, m))
                k = int(rng.integers(0, 3))
                if k == 0:
                    p[i, pos] = np.frombuffer(b"ACGTN", np.uint8)[rng.integers(0, 5)]
                elif k == 1:
                    p[i, pos:] = np.roll(p[i, pos:], 1)
                else:
                    p[i, pos:] = np.roll(p[i, pos:], -1)
        d = gpu.banded_edit_distance_batch(t, p, e)
        packed = reference.pack(t, p)
        try:
            ref = packed.banded(e)
        finally:
            packed.free()
        assert (d == ref).all(), (m, e, np.nonzero(d != ref)[0][:5])


def test_acceptance_criterion2_oracle_on_gpu(gpu, oracle):
    z = np.load(os.path.join(ROOT, "tests", "golden", "fr_m100_e2.npz"))
    t, p = oracle.generate_pairs(int(z["seed"]), 100_000, 100, 0, 2)
    d = gpu.banded_edit_distance_batch(t, p, 2)
    assert ((d >= 0) == z["similar"]).all()


def run(*args, stdin=None):
    r = subprocess.run([CLI, *args], input=stdin, capture_output=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def test_cli_filter_matches_oracle(gpu, oracle, tmp_path):
    t, p = oracle.generate_pairs(77, 20000, 100, 0, 10)
    f = tmp_path / "pairs.tsv"
    f.write_bytes(b"".join(t[i].tobytes() + b"\t" + p[i].tobytes() + b"\n" for i in range(len(t))))
    rc, out, err = run("filter", "--pairs", str(f), "--e", "5", "--verbose")
    assert rc == 0, err
    acc, est, _ = oracle.shouji_batch(t, p, 5)
    bits = np.unpackbits(acc.view(np.uint8), bitorder="little")[:len(t)]
    expect = b"".join(b"%d\t%d\n" % (bits[i], est[i]) for i in range(len(t)))
    assert out == expect
    rep = json.loads(err)
    assert list(rep) == ["command", "algo", "width", "m", "source", "e", "total", "accepted",
                         "rejected"]
    assert rep["accepted"] == int(bits.sum()) and rep["total"] == 20000 and rep["m"] == 100
    # --threads never changes a byte (acceptance_tests.cpp:317-341)
    rc2, out2, err2 = run("filter", "--pairs", str(f), "--e", "5", "--verbose", "--threads", "8")
    assert rc2 == 0 and out2 == out and err2 == err
    # stdin input and --e-percent (floored): 5.9% of 100 -> 5
    rc3, out3, err3 = run("filter", "--pairs", "-", "--e-percent", "5.9", "--verbose",
                          stdin=f.read_bytes())
    assert rc3 == 0 and out3 == out and json.loads(err3)["e"] == 5


def test_cli_filter_generator_and_oracle_algo(gpu, oracle, reference):
    rc, out, err = run("filter", "--seed", "3", "--count", "5000", "--len", "100", "--e", "3",
                       "--algo", "oracle", "--verbose")
    assert rc == 0, err
    t, p = oracle.generate_pairs(3, 5000, 100, 0, 6)  # default edits 0..2e
    packed = reference.pack(t, p)
    try:
        d = packed.banded(3)
    finally:
        packed.free()
    expect = b"".join((b"1\t%d\n" % x) if x >= 0 else b"0\t-\n" for x in d)
    assert out == expect


def test_cli_eval_counts(gpu, oracle, reference):
    rc, out, err = run("eval", "--seed", "1105", "--count", "100000", "--len", "100", "--edits",
                       "0..5", "--e", "5")
    assert rc == 0, err
    rep = json.loads(err)
    t, p = oracle.generate_pairs(1105, 100000, 100, 0, 5)
    packed = reference.pack(t, p)
    try:
        acc, _, _ = packed.shouji(5)
        d = packed.banded(5)
    finally:
        packed.free()
    a = np.unpackbits(acc.view(np.uint8), bitorder="little")[:100000].astype(bool)
    within = d >= 0
    assert rep["oracle_accepted"] == int(within.sum())
    assert rep["filter_accepted"] == int(a.sum())
    assert rep["falsely_rejected"] == int((within & ~a).sum()) == 41  # proj/test_output.txt:11
    assert rep["falsely_accepted"] == int((~within & a).sum())


def test_cli_bench_runs(gpu):
    rc, out, err = run("bench", "--len", "100,200", "--e", "2,5", "--count", "50000",
                       "--repeats", "2")
    assert rc == 0, err
    lines = out.decode().splitlines()
    assert lines[0].startswith("algo,m,e,count,repeats,median_seconds")
    assert len([l for l in lines if l.startswith("shouji,")]) == 4 + 2


def test_cli_magnet_filter_and_eval(gpu, oracle, reference):
    """--algo magnet routes filter/eval/bench through pf_magnet_filter_batch (run_filter's
    other branch, evaluate.cpp:13-21)."""
    rc, out, err = run("filter", "--seed", "5", "--count", "6000", "--len", "150", "--e", "7",
                       "--algo", "magnet", "--verbose")
    assert rc == 0, err
    t, p = oracle.generate_pairs(5, 6000, 150, 0, 14)
    acc, est = reference.magnet_batch(t, p, 7)
    bits = np.unpackbits(acc.view(np.uint8), bitorder="little")[:6000]
    assert out == b"".join(b"%d\t%d\n" % (bits[i], est[i]) for i in range(6000))
    assert json.loads(err)["algo"] == "magnet"
    rc, out, err = run("eval", "--seed", "1105", "--count", "20000", "--len", "100", "--edits",
                       "0..5", "--e", "5", "--algo", "magnet")
    assert rc == 0, err
    rep = json.loads(err)
    t, p = oracle.generate_pairs(1105, 20000, 100, 0, 5)
    acc, _ = reference.magnet_batch(t, p, 5)
    packed = reference.pack(t, p)
    try:
        d = packed.banded(5)
    finally:
        packed.free()
    a = np.unpackbits(acc.view(np.uint8), bitorder="little")[:20000].astype(bool)
    within = d >= 0
    assert rep["filter_accepted"] == int(a.sum())
    assert rep["falsely_rejected"] == int((within & ~a).sum())
    assert rep["falsely_accepted"] == int((~within & a).sum())
    rc, out, err = run("bench", "--len", "100", "--e", "5", "--count", "20000", "--repeats", "1",
                       "--algo", "magnet")
    assert rc == 0, err
    assert out.decode().splitlines()[1].startswith("magnet,100,5,20000,1,")
    rc, _, err = run("filter", "--seed", "5", "--count", "10", "--len", "10", "--e", "1",
                     "--algo", "nope")
    assert rc == 1 and b"--algo" in err  # usage errors exit 1 (cli.cpp:357-359)
