"""The reference's pybind11 module (python/module.cpp), compiled UNMODIFIED
against include/octohull and linked to libocto_b200.so (oracle/Makefile
`pymodule`), driven through the checks of the reference's Python smoke
tests (tests/python/test_smoke.py:17-60)."""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

MOD_DIR = os.path.join(ROOT, "oracle", "_ref", "pymodule")


@pytest.fixture(scope="module")
def core():
    if not any(f.startswith("_core") for f in os.listdir(MOD_DIR)) if os.path.isdir(MOD_DIR) else True:
        pytest.skip("relinked reference module not built (needs /root/reference at build time)")
    sys.path.insert(0, MOD_DIR)
    try:
        return importlib.import_module("_core")
    finally:
        sys.path.remove(MOD_DIR)


def cycles_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and any(np.array_equal(np.roll(b, -s, axis=0), a)
                                      for s in range(len(a)))


def test_generate_and_errors(core, oracle):
    a = core.generate("normal", 500, seed=3)
    assert np.array_equal(a, core.generate("normal", 500, seed=3))
    assert np.array_equal(a, oracle.generate("normal", 500, 3))
    with pytest.raises(ValueError):
        core.generate("triangle", 10)
    with pytest.raises(ValueError):
        core.generate("normal", 10, distort=2.0)


@pytest.mark.gpu
def test_smoke_checks_on_b200(core, oracle):
    pts = np.array([[0, 0], [1, 0], [1, 1], [0, 1], [0.5, 0.5]], dtype=float)
    hull = core.heaphull(pts)
    assert hull.shape == (4, 2) and cycles_equal(hull, core.monotone_chain(pts))
    disk = core.generate("disk", 2000, seed=7)
    assert cycles_equal(core.heaphull(disk), core.monotone_chain(disk))
    normal = core.generate("normal", 10000, seed=11)
    labels = core.classify(normal)
    assert labels.shape == (10000,) and float((labels == 0).mean()) >= 0.995
    assert np.array_equal(labels, oracle.classify(normal))
    circ = core.generate("circle", 3000, seed=5, distort=2.0)
    assert np.array_equal(core.heaphull(circ, threads=1), core.heaphull(circ, threads=4))
    assert np.array_equal(core.classify(circ, threads=1, chunk=1),
                          core.classify(circ, threads=4, chunk=1024))
    assert np.array_equal(core.heaphull(circ), oracle.heaphull(circ))
    with pytest.raises(ValueError):
        core.heaphull(np.zeros((3, 3)))
