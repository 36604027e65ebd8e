"""The reference arm of bench.py (`--impl reference`) on the CPU: it times the
unmodified reference package staged under baseline/_ref through its own
public API (ttpar.round_tt(serial_tt(X)), parallel.py:293) when that install
is present, and the oracle port otherwise; either way the JSON line carries
the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_cfg1():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["config"]["same_config"] is True
    staged = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "ttpar"))
    assert line["cpu_baseline"]["kind"] == ("reference" if staged else "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
