"""bench.py's reference arm on CPU: it runs only the unmodified reference
library (oracle/_ref) and never maps the product library librunq_b200.so —
the driver's reference ratio is void otherwise."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload", ["c1", "c2", "c3", "q1", "q6", "c5"])
def test_reference_arm_does_not_load_product(ref, workload):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
                          "--rows", "2000000", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["product_library_loaded"] is False
    assert line["cpu_baseline"]["kind"] == "reference" and line["value"] > 0
