"""bench.py's contract on the GPU at a reduced size: the single-GPU JSON line (keys the driver
reads, e2e with its copies, roofline, launches) and the multi-rank path (`--gpus 2` re-launched
under torch.distributed.run; both ranks pinned to device 0 with PF_BENCH_DEVICE and a gloo
process group, which exercises the rank plumbing, the max-over-ranks timing and the whole-job
value — the timing itself is meaningless with two ranks on one GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _run(args, env_extra=None, timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    j = _run(["--steps", "3", "--warmup", "3", "--pairs", "2000000", "--no-cpu"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "e2e", "gpu_launches",
              "clocks"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 3 and j["value"] > 1e9
    assert j["gpu_launches"] >= 2 * 3  # pack + search per timed step
    assert j["roofline"]["unit"] == "GB/s" and 0 < j["roofline"]["frac"] < 1.2
    e2e = j["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0 and e2e["value"] > 0


def test_bench_two_ranks_plumbing():
    j = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--pairs", "1000000", "--no-cpu",
              "--no-e2e"], env_extra={"PF_BENCH_DEVICE": "0", "PF_DIST_BACKEND": "gloo"})
    assert j["n_gpus"] == 2
    assert j["config"]["global_pairs"] == 2 * 1000000
    # whole-job value = pairs of all ranks / max-over-ranks step time
    assert abs(j["value"] - 2 * 1000000 / (j["ms_per_step"] * 1e-3)) < 1e-6 * j["value"]


def test_bench_reference_arm_line():
    """`--impl reference`: the reference library on the host cores over a prefix of the same
    configs[1] bytes, the same metric/config keys, e2e with no device copies."""
    j = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], timeout=900)
    assert j["impl"] == "reference"
    ours = _run(["--steps", "3", "--warmup", "3", "--pairs", "2000000", "--no-cpu", "--no-e2e"])
    assert j["metric"] == ours["metric"] and j["unit"] == ours["unit"]
    assert j["value"] > 0 and j["cpu_baseline"]["kind"] in ("reference", "port")
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
