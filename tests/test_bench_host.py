"""Host logic of bench.py (no GPU): the reference arm's host-RAM guard and its JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_oracle_fits_reports_state_size():
    # 2^40 complex128 amplitudes = 16 TiB: more than any host here
    why = bench.oracle_fits({"n": 40})
    assert why is not None and "16384 GiB" in why
    assert bench.oracle_fits({"n": 10}) is None


def test_reference_arm_line_small_workload():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "qv28", "--steps", "1", "--warmup", "3", "--ref-step-s", "0.5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" not in line:
        assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
        assert line["e2e"]["h2d_bytes_per_step"] == 0
