"""The C++ drop-in's overlapped path (shim/blockcells_b200_shim.cpp run_gpu):
batches of >= 16384 independent groups are solved in four group-aligned
pieces while the host packs the next piece and unpacks the previous one.
Every output bit -- x of every cell, per-group iterations, the report's max
rms, effective and summed iterations (tests/cpp/dropin_bench.cpp's digest) --
must equal the single-call path's (BLOCKCELLS_B200_OVERLAP=0), as
merge_groups (strategies.cpp:71-87) folds groups independently of how the
batch is split."""
import json
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin", "dropin_bench")


def run(cells, algo, overlap, h, tol, max_iter):
    env = dict(os.environ, BLOCKCELLS_B200_OVERLAP=overlap, BLOCKCELLS_B200_ALGO=algo)
    r = subprocess.run([BIN, str(cells), "1", "0", "156", repr(h), repr(tol), str(max_iter)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp binaries not built (needs /root/reference at build time)")
@pytest.mark.parametrize("algo,cells,regime", [("bicgstab", 20011, "C"), ("bicg", 16384, "C"), ("bicgstab", 17000, "P")])
def test_overlapped_pieces_equal_one_call(algo, cells, regime):
    h, tol, max_iter = (1.0, 1e-10, 1000) if regime == "C" else (120.0, 1e-30, 60)
    one = run(cells, algo, "0", h, tol, max_iter)
    pieces = run(cells, algo, "1", h, tol, max_iter)
    assert one["output_digest"] == pieces["output_digest"]
    assert one["iterations_sum"] == pieces["iterations_sum"]
    assert one["breakdown_fallbacks"] == pieces["breakdown_fallbacks"]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp binaries not built (needs /root/reference at build time)")
@pytest.mark.parametrize("overlap", ["0", "1"])
@pytest.mark.parametrize("bad,want", [
    ({"DROPIN_BAD_PATTERN_CELL": "19000"}, "batched system: cells do not share one sparsity pattern"),
    ({"DROPIN_BAD_RHS_CELL": "5"}, "batched system: rhs dimension"),
    # check() tests every matrix before any rhs: the later pattern error wins
    ({"DROPIN_BAD_PATTERN_CELL": "19000", "DROPIN_BAD_RHS_CELL": "5"},
     "batched system: cells do not share one sparsity pattern"),
])
def test_overlapped_pieces_raise_check_errors(overlap, bad, want):
    """The piecewise pattern check throws BatchedSystem::check's exception
    (strategies.cpp:91-107) for the lowest bad cell, with check()'s precedence."""
    env = dict(os.environ, BLOCKCELLS_B200_OVERLAP=overlap, BLOCKCELLS_B200_ALGO="bicgstab", **bad)
    r = subprocess.run([BIN, "20000", "1", "0", "156", "1.0", "1e-10", "50"], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["error"] == want


WS_B200 = os.path.join(os.path.dirname(BIN), "ws_dump_b200")
WS_REF = os.path.join(os.path.dirname(BIN), "ws_dump_reference")


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.exists(WS_B200) and os.path.exists(WS_REF)),
                    reason="tests/cpp binaries not built (needs /root/reference at build time)")
def test_bicg_workspace_outputs_equal_reference():
    """bicg_solve(..., BicgWorkspace& ws) (bicg.hpp:42-48): x, iterations,
    flags, final rms and ws.per_block_error (the per-block partials of the
    final fresh residual, bicg.cpp:61-72) bit for bit, drop-in vs the
    reference's own bicg.o, on one- and multi-block reduction plans, converged
    and iteration-capped solves (tests/cpp/ws_dump.cpp)."""
    ref = subprocess.run([WS_REF], capture_output=True, text=True, timeout=600)
    got = subprocess.run([WS_B200], capture_output=True, text=True, timeout=600)
    assert ref.returncode == 0 and got.returncode == 0, got.stderr[-2000:] + ref.stderr[-2000:]
    assert ref.stdout.count("per_block_error") == 10
    assert got.stdout == ref.stdout
