"""bench.py's JSON-line contract on CPU: the reference arm (the oracle, the only place besides
tests / smoke / cpu_baseline that runs it) prints one line with the base contract's keys plus
impl / cpu_baseline / e2e; an N > 1 request outside torchrun prints an error line; datagen's
instances reproduce its labels."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=600, env=env)
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    return r.returncode, json.loads(lines[-1]) if lines else None


def test_reference_arm_line():
    rc, d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert rc == 0 and d is not None
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_pgm_workload():
    rc, d = run_bench("--impl", "reference", "--workload", "c6", "--steps", "1", "--warmup", "0")
    assert rc == 0 and d["impl"] == "reference" and "PGM" in d["config"]["workload"]


def test_multi_gpu_needs_torchrun():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    rc, d = run_bench("--gpus", "2", "--steps", "1", "--warmup", "0", env=env)
    assert rc != 0 and "error" in d


def test_instances_reproduce_labels():
    """datagen.instances are the draws behind datagen.labels (same seeds): the actionness label
    is positive exactly on snippets that overlap an instance."""
    sys.path.insert(0, ROOT)
    import datagen
    B, T = 6, 100
    lab = datagen.labels(B, T, rank=1, batch_idx=3)
    seg, cnt = datagen.instances(B, T, rank=1, batch_idx=3)
    for v in range(B):
        cover = np.zeros(T, bool)
        for i in range(cnt[v]):
            s, e = seg[v, i]
            t = np.arange(T)
            cover |= (np.minimum(t + 1, e) - np.maximum(t, s)) > 1e-6
        assert np.array_equal(lab[v, 0] > 0, cover), v
