"""bench.py's host-side parts on CPU: the reference arm (the oracle timed as it stands) prints the
contract's JSON line, and the algorithmic-bytes model matches hand counts."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"]
    assert line["steps"] == 3 and line["warmup"] == 3 and line["n_gpus"] == 1
    assert line["metric"].startswith("verified tokens/s")
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"].startswith("c1")


def test_algorithmic_bytes_by_hand():
    """Sampled: rows 0..L of p and of q (q has no row k), plus the k ids and k+2 output words;
    greedy: p rows only."""
    import bench
    V, k, e = 1000, 4, 4
    # L = 0: p_0 and q_0; L = 2: p_0..p_2 and q_0..q_2; L = k: p_0..p_4 and q_0..q_3
    want = [2 * V * e, 6 * V * e, 9 * V * e]
    got = bench.algorithmic_bytes(np.array([0, 2, 4]), V, k, e, False) - (4 * k + 4 * (k + 2))
    assert list(got) == want
    got = bench.algorithmic_bytes(np.array([0, 2, 4]), V, k, e, True) - (4 * k + 4 * (k + 2))
    assert list(got) == [1 * V * e, 3 * V * e, 5 * V * e]
