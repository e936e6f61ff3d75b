"""bench.py's reference arm on CPU: the reference's own generator and
heaphull_run only (nothing of the product library loaded), and the same
`config` as the B200 arm for the same flags."""

import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def _ref_available():
    from oracle import Reference
    return Reference.available()


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
def test_reference_arm_loads_only_the_reference():
    probe = (
        "import sys, runpy, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--points', '200000', '--steps', '2',"
        " '--warmup', '1']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "mods = [m for m in sys.modules if m.startswith('paper_2209_12310_b200')]\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'mods': mods, 'so': 'libocto_b200' in maps}))\n")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    line, probe_out = lines[-2], lines[-1]
    assert probe_out == {"mods": [], "so": False}
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"

    import bench
    sys.argv = ["bench.py", "--points", "200000"]
    assert line["config"] == bench.config(bench.parse(), 1)


def test_job_corpus_and_shards():
    import bench
    sys.argv = ["bench.py"]
    a = bench.parse()
    assert bench.job(a, 1)["total"] == 1_000_000_000
    j = bench.job(a, 8)
    assert j["total"] == 4_000_000_000 and j["scaling"] == "strong"
    spans = [bench.shard_of(j["total"], 8, r) for r in range(8)]
    assert spans[0][0] == 0 and sum(c for _, c in spans) == j["total"]
    assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(7))
    sys.argv = ["bench.py", "--weak"]
    assert bench.job(bench.parse(), 4)["total"] == 4_000_000_000
    assert bench.config(a, 1)["workload"].startswith("BASELINE configs[2]")
    assert bench.config(a, 8)["workload"].startswith("BASELINE configs[4]")
