"""CPU: the synthetic workload generator reproduces the reference's
generate_mechanism / newton_system bit for bit."""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import oracle_ffi as of
from paper_2405_17363_b200 import Mechanism

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "workload_digests.txt")


def digests():
    with open(GOLD) as f:
        return dict(line.split() for line in f if line.strip())


@pytest.mark.parametrize("species", [156, 312])
def test_generator_matches_golden_digests(species):
    d = digests()
    m = Mechanism(species, 3 * species, 0)
    assert hashlib.sha256(m.row_ptr.tobytes() + m.col_idx.tobytes()).hexdigest() == d[f"m{species}_pattern"]
    for h in (120.0, 1.0):
        v, b = m.newton_batch(37, 10, 1000, h)
        assert hashlib.sha256(v.tobytes() + b.tobytes()).hexdigest() == d[f"m{species}_h{int(h)}"]


def test_m156_shape():
    m = Mechanism(156, 468, 0)
    assert m.nnz == 1556
    lens = np.diff(m.row_ptr)
    assert lens.min() == 2 and lens.max() == 24
    assert Mechanism(312, 936, 0).nnz == 3032


@pytest.mark.skipif(not of.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("species,seed,mode,h", [(156, 0, 1, 120.0), (156, 0, 0, 1.0), (40, 3, 1, 1.0),
                                                 (312, 1, 1, 120.0)])
def test_generator_bitwise_vs_reference(species, seed, mode, h):
    m = Mechanism(species, 3 * species, seed)
    v, b = m.newton_batch(100, 20, 1000, h, mode)
    v2 = np.zeros_like(v)
    b2 = np.zeros_like(b)
    assert of.ref().ref_newton_batch(species, 3 * species, seed, 100, 20, 1000, mode, h, of.ptr(v2), of.ptr(b2)) == 0
    np.testing.assert_array_equal(of.bits(v), of.bits(v2))
    np.testing.assert_array_equal(of.bits(b), of.bits(b2))


def test_threads_do_not_change_values():
    m = Mechanism(156, 468, 0)
    v1, b1 = m.newton_batch(0, 64, 64, 120.0, threads=1)
    v8, b8 = m.newton_batch(0, 64, 64, 120.0, threads=8)
    np.testing.assert_array_equal(of.bits(v1), of.bits(v8))
    np.testing.assert_array_equal(of.bits(b1), of.bits(b8))
