"""The reference's own test programs, UNMODIFIED, compiled by oracle/Makefile
(`reftests`) against this library's drop-in headers and linked to
libocto_b200.so: the unit suites tests/test_{geometry,parallel,pointgen,io,
filter,hull,bench}.cpp of /root/reference/proj, the CLI
tools/octohull_main.cpp (against a CLI11 shim) and the acceptance harness
tests/acceptance.cpp (criteria 1-9, the CLI among them).  geometry /
parallel / pointgen / io and the CLI's generate exercise host code only;
filter, hull, bench and acceptance drive the sm_100a kernels."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "reftests")


def run_suite(name):
    path = os.path.join(BIN, f"test_{name}")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    summary = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert r.returncode == 0, r.stderr[-4000:] + summary
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| 0 failed", summary)
    assert m and m.group(1) == m.group(2), summary


@pytest.mark.parametrize("suite", ["geometry", "parallel", "pointgen", "io"])
def test_reference_host_suites(suite):
    run_suite(suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["filter", "hull", "bench"])
def test_reference_gpu_suites(suite):
    run_suite(suite)


def _cli():
    path = os.path.join(BIN, "octohull_cli")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    return path


def test_reference_cli_host_commands(tmp_path):
    # generate + the parse errors need no device
    cli = _cli()
    out = tmp_path / "p.txt"
    r = subprocess.run([cli, "generate", "--dist", "disk", "--n", "1000", "--seed", "9",
                        "--out", str(out)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "wrote 1000 points" in r.stdout, r.stderr
    assert len(out.read_text().splitlines()) == 1000
    r = subprocess.run([cli, "hull", "--algo", "heaphull"], capture_output=True, text=True,
                       timeout=60)
    assert r.returncode != 0  # --in is required (acceptance criterion 9)
    r = subprocess.run([cli, "bench", "--dist", "normal", "--n-list", "10", "--reps", "0"],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode != 0  # --reps must be positive


@pytest.mark.gpu
def test_reference_acceptance_criteria(tmp_path):
    # acceptance.cpp with the reference CLI (built against this library) as
    # its CLI: every criterion must print [PASS]
    acc = os.path.join(BIN, "acceptance")
    if not os.path.exists(acc):
        pytest.skip(f"{acc} not built (needs /root/reference at build time)")
    r = subprocess.run([acc, _cli(), str(tmp_path / "scratch")], capture_output=True,
                       text=True, timeout=1800)
    out = r.stdout
    assert out.count("[PASS]") == 9 and "[FAIL]" not in out, out[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0
