"""bench.py contract checks that need no GPU: both arms print BASELINE.json's metric string (so
the driver can pair them), and `--gpus 2` without torchrun re-launches itself with two ranks
(the reference arm runs on rank 0 only and reports n_gpus 2)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_metric_is_baselines():
    sys.path.insert(0, ROOT)
    src = open(os.path.join(ROOT, "bench.py")).read()
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert f'METRIC = "{base["metric"]}"' in src
    assert src.count('"metric": METRIC') == 2  # the bsra arm and the reference arm


def test_reference_arm_two_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], cwd=ROOT, stdout=subprocess.PIPE,
                       stderr=subprocess.DEVNULL, timeout=600)
    assert r.returncode == 0
    lines = [l for l in r.stdout.decode().splitlines() if l.strip()]
    assert len(lines) == 1, lines
    out = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["metric"] == base["metric"]
    assert out["cpu_baseline"]["kind"] == "oracle" and out["e2e"]["h2d_bytes_per_step"] == 0
