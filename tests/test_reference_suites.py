"""The reference's own unit suites (tests/test_{geometry,parallel,pointgen,
io,filter,hull}.cpp of /root/reference/proj), UNMODIFIED, compiled by
oracle/Makefile (`reftests`) against this library's drop-in headers and
linked to libocto_b200.so.  geometry / parallel / pointgen / io exercise
host code only; filter and hull drive the sm_100a kernels and need the GPU."""

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
@pytest.mark.parametrize("suite", ["filter", "hull"])
def test_reference_gpu_suites(suite):
    run_suite(suite)
