"""bench.py's reference arm (--impl reference) runs on the CPU: its JSON line
carries the keys the driver reads (impl, metric, value, unit, e2e with zero
copy bytes, cpu_baseline with kind/cores/sample), on the same metric as the
B200 arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as of
    if not (of.have_ref() or os.path.exists(of.ORC_PATH)):
        pytest.skip("no CPU checker built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--cells", "300", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("BiCGSTAB cell-solves/sec") and line["unit"] == "cell-solves/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    assert line["ms_per_step"] > 0 and line["steps"] == 1
    # the same config dict the B200 arm prints for the same flags (the driver's same_config)
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    from paper_2405_17363_b200 import REGIME_P
    args = argparse.Namespace(algo="bicgstab", strategy="block-cells-1")
    assert line["config"] == bench.bench_config(args, 156, 1556, 300, 300, REGIME_P, 1)
    # the stock reference algorithm is timed beside the composed BiCGSTAB
    assert line["reference_bicg"]["value"] > 0
