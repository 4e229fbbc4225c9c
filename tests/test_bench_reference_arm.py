"""bench.py's reference arm (CPU only): the reference's algorithm on the
host through oracle/ alone -- no module of the product package may be
imported on that arm -- printing one valid JSON line."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1"]
sys.path.insert(0, {repo!r})
import bench
bench.main()
loaded = sorted(m for m in sys.modules if m.startswith("paper_2208_11469_b200"))
print("LOADED=" + json.dumps(loaded))
"""


def test_reference_arm_runs_without_product_package():
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(repo=REPO)], capture_output=True,
                         text=True, timeout=600, cwd=REPO, env=dict(os.environ, WORLD_SIZE="1"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = out.stdout.splitlines()
    rec = json.loads(next(ln for ln in lines if ln.startswith("{")))
    loaded = json.loads(next(ln for ln in lines if ln.startswith("LOADED="))[len("LOADED="):])
    assert loaded == [], loaded
    assert rec["impl"] == "reference" and rec["n_gpus"] == 1
    for key in ("metric", "value", "unit", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in rec, key
    assert rec["value"] > 0 and rec["cpu_baseline"]["kind"] == "port"
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["e2e"]["value"] == rec["value"]
    assert rec["config"]["m"] == 15702278  # R-MAT s20 seed 1 from the oracle's generator
