"""Random batched systems in the style of the reference's test fixtures
(tests/test_util.hpp:15-79, tests/test_strategies.cpp:18-50): one shared
sparsity pattern, per-cell strictly diagonally dominant values.  numpy's
generator replaces mt19937_64: both sides of every comparison see the same
arrays, so the stream itself does not matter."""
from __future__ import annotations

import numpy as np


def random_pattern(rng: np.random.Generator, n: int, density: float = 0.3):
    rows, cols = [], []
    for i in range(n):
        for j in range(n):
            if i == j or rng.random() < density:
                rows.append(i)
                cols.append(j)
    row_ptr = np.zeros(n + 1, np.int32)
    for r in rows:
        row_ptr[r + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    return row_ptr, np.array(cols, np.int32)


def random_batch(rng: np.random.Generator, cells: int, species: int, density: float = 0.3,
                 row_ptr=None, col_idx=None):
    if row_ptr is None:
        row_ptr, col_idx = random_pattern(rng, species, density)
    nnz = int(row_ptr[-1])
    values = np.empty((cells, nnz))
    for c in range(cells):
        for i in range(species):
            lo, hi = row_ptr[i], row_ptr[i + 1]
            off = col_idx[lo:hi] != i
            v = rng.uniform(-1.0, 1.0, hi - lo)
            v[~off] = np.abs(v[off]).sum() + 1.0 + rng.random()
            values[c, lo:hi] = v
    rhs = rng.uniform(-1.0, 1.0, (cells, species))
    return row_ptr, col_idx, values, rhs
