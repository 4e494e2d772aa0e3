"""CLI caller timing: `shouji-b200 gen` a TSV of N pairs (m=100, edits 0..10) into
/tmp, then time `filter --pairs FILE --e 5` (load + GPU validation + filter +
output) next to `cat FILE`. python tools/exp_cli_filter.py [N]"""
import os
import subprocess
import sys
import time

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1809_07858_b200", "shouji-b200")
path = "/tmp/exp_cli_pairs.tsv"


def timed(cmd):
    t0 = time.perf_counter()
    subprocess.run(cmd, shell=True, check=True)
    return time.perf_counter() - t0


if not os.path.exists(path) or os.path.getsize(path) != N * 202:
    timed(f"{CLI} gen --count {N} --len 100 --edits 0..10 --pairs {path}")
cat = timed(f"cat {path} > /dev/null")
runs = [timed(f"{CLI} filter --pairs {path} --e 5 > /tmp/exp_cli_out.txt 2>/dev/null") for _ in range(3)]
print(f"pairs {N}: cat {cat:.2f} s, filter {min(runs):.2f} s = {N / min(runs) / 1e6:.1f} M pairs/s")

# phase split through the Python mirror (same C ABI calls as the CLI)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_07858_b200 as pf  # noqa: E402

t0 = time.perf_counter()
ds = pf.load_pairs_file(path)
t1 = time.perf_counter()
acc, est, _ = pf.shouji_filter_batch(ds.text(), ds.pattern(), 5, estimates=True)
t2 = time.perf_counter()
print(f"load_pairs_file {t1 - t0:.2f} s, filter batch {t2 - t1:.3f} s")
