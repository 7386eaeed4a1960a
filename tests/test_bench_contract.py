"""bench.py's reference arm runs on the host cores only (the CPU oracle), so its JSON line can be
checked here: one line, the contract's keys, the oracle as the baseline kind."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "products-shaped"


def test_ring_plan_fits_memory():
    # the timed output ring: one slot per step, capped at 4 GB and at the HBM left after the store
    import bench

    slot = 8192 * 4 * 100 * 2  # products bf16 batch: 6.55 MB
    assert bench.ring_plan(299, 8, slot, free_bytes=150e9) == 299  # whole epoch fits under the cap
    assert bench.ring_plan(1695, 8, slot, free_bytes=150e9) == int(4e9 // slot)  # 4 GB cap
    tight = (2 << 30) + 20 * slot
    assert bench.ring_plan(1695, 8, slot, free_bytes=tight) == 20  # what is left after the reserve
    assert bench.ring_plan(1695, 8, slot, free_bytes=1e9) == 8  # never below one launch's worth
    assert bench.ring_plan(3, 8, slot, free_bytes=150e9) == 3
