"""bench.py's contract pieces that run without a GPU: the reference arm (the
oracle on the host, its JSON line) and the e2e object's construction."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "0", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, r.stdout  # exactly one JSON line on stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "points/s"
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0
    assert e["d2h_bytes_per_step"] == 0 and e["unit"] == d["unit"]


def test_e2e_line_prefers_the_pipelined_stream():
    import bench
    e = bench.e2e_line(1000, 10, 1, 5.0e5, 0.05, 0.004, 123)
    assert e["mode"] == "pipelined" and math.isclose(e["value"], 1000 * 10 / 0.004)
    assert e["synchronous_value"] == 5.0e5
    assert math.isclose(e["synchronous_wall_value"], 1000 * 10 / 0.05)
    assert e["h2d_bytes_per_step"] == 16 * 1000 and e["d2h_bytes_per_step"] == 123
    # no pipelined run (rolling map): the synchronous number is the value
    e = bench.e2e_line(1000, 10, 2, 5.0e5, 0.05, float("nan"), 123)
    assert e["mode"] == "synchronous" and e["value"] == 5.0e5
