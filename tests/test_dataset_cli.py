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


# --- TSV ingest on the host cores (pf_dataset_load_tsv_file; no CUDA context) -------

def _load_file(path):
    import ctypes as C
    from paper_1809_07858_b200 import _lib as L
    h = C.c_void_p()
    err = L.PfError()
    st = L.lib.pf_dataset_load_tsv_file(None, str(path).encode(), C.byref(h), C.byref(err))
    if st != L.PF_OK:
        return st, err, None
    n, m = L.lib.pf_dataset_size(h), L.lib.pf_dataset_length(h)
    t = np.frombuffer((C.c_uint8 * (n * m)).from_address(L.lib.pf_dataset_text(h)), np.uint8).reshape(n, m).copy()
    p = np.frombuffer((C.c_uint8 * (n * m)).from_address(L.lib.pf_dataset_pattern(h)), np.uint8).reshape(n, m).copy()
    L.lib.pf_dataset_free(h)
    return st, err, (t, p)


def test_load_tsv_file_roundtrip_and_edges(oracle, tmp_path):
    # load_pairs_file (dataset.cpp:13-44): mmap'd regular file, getline line semantics
    t, p = oracle.generate_pairs(11, 5000, 100, 0, 10)
    body = b"".join(t[i].tobytes() + b"\t" + p[i].tobytes() + b"\n" for i in range(len(t)))
    f = tmp_path / "pairs.tsv"
    f.write_bytes(body)
    st, _, rec = _load_file(f)
    assert st == 0 and (rec[0] == t).all() and (rec[1] == p).all()
    f.write_bytes(body[:-1])  # no trailing newline: the last line still counts
    st, _, rec = _load_file(f)
    assert st == 0 and rec[0].shape == (5000, 100) and (rec[1] == p).all()
    f.write_bytes(b"")  # empty input
    st, err, _ = _load_file(f)
    assert st != 0 and err.line == 1 and b"no pairs in input" in bytes(err.message)
    bad = bytearray(body)
    bad[3 * 202 + 101 + 17] = ord("x")  # line 4, pattern position 17
    f.write_bytes(bytes(bad))
    st, err, _ = _load_file(f)
    assert st != 0 and err.line == 4 and err.position == 17 and err.byte == ord("x")
    assert b"illegal character 'x' at position 17" in bytes(err.message)
    extra = body[:202 * 7] + t[7].tobytes() + b"\t" + p[7].tobytes() + b"\tX\n"
    f.write_bytes(extra)
    st, err, _ = _load_file(f)
    assert st != 0 and err.line == 8 and b"found more" in bytes(err.message)
    st, err, _ = _load_file(tmp_path / "missing.tsv")
    assert st != 0 and b"cannot open pair file" in bytes(err.message)


def test_load_tsv_from_a_fifo(oracle, tmp_path):
    # a non-regular file (named pipe) is read to its end instead of mapped
    import threading
    t, p = oracle.generate_pairs(12, 300, 50, 0, 5)
    body = b"".join(t[i].tobytes() + b"\t" + p[i].tobytes() + b"\n" for i in range(len(t)))
    fifo = tmp_path / "pairs.fifo"
    os.mkfifo(fifo)
    w = threading.Thread(target=lambda: fifo.write_bytes(body))
    w.start()
    st, _, rec = _load_file(fifo)
    w.join()
    assert st == 0 and (rec[0] == t).all() and (rec[1] == p).all()


def test_load_tsv_line_beyond_length_limit(tmp_path):
    # A well-formed first line the reference would load, with records longer than this
    # implementation's m < 2^24 limit: reported as an invalid parameter with its own
    # message, not as a length mismatch of the line against itself.
    from paper_1809_07858_b200 import _lib as L
    k = 1 << 24
    f = tmp_path / "long.tsv"
    f.write_bytes(b"A" * k + b"\t" + b"C" * k + b"\n")
    st, err, _ = _load_file(f)
    assert st == L.PF_ERR_INVALID_PARAMETERS and err.line == 1
    assert b"exceeds the supported maximum" in bytes(err.message)
    assert b"length mismatch" not in bytes(err.message)
