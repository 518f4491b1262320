"""CPU: the C-ABI libraries load without a GPU and export every symbol the
headers declare; the host-side planning and the fused kernel's SpMV
schedule / reduction geometry reproduce the reference's arithmetic order
(emulated here in exact IEEE double arithmetic, no GPU needed)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_ffi as of
from fixtures import random_batch
from paper_2405_17363_b200 import Mechanism, _native
from paper_2405_17363_b200._native import SolveParams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bcw?_[a-z_0-9]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("blockcells_b200.h", "b200"), ("blockcells_workload.h", "workload")])
def test_library_exports_every_declared_symbol(header, lib):
    dll = getattr(_native, lib)()
    names = declared(header)
    assert len(names) >= 6
    missing = [n for n in names if not hasattr(dll, n)]
    assert not missing, missing


def test_kernels_are_sm100a():
    """The library carries sm_100a SASS (cuobjdump), with no FMA in the solver."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _native.LIB_B200], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", _native.LIB_B200], capture_output=True, text=True).stdout
    assert "block_cells_kernel" in sass and "DADD" in sass and "DMUL" in sass


def plan(species, strategy, k, cells, mtpb=1024):
    prm = SolveParams()
    prm.strategy, prm.cells_per_block, prm.cells, prm.max_threads_per_block = strategy, k, cells, mtpb
    prm.tol, prm.max_iter = 1e-8, 10
    ng, cpb = C.c_int64(), C.c_double()
    st = _native.b200().bc_plan(species, C.byref(prm), C.byref(ng), C.byref(cpb))
    return st, ng.value, cpb.value


def test_plan_mirrors_plan_kernel():
    """exec_model.cpp:102-161 + strategies.cpp:209-213 (same as the oracle)."""
    for species in (1, 13, 156, 312, 1024):
        for cells in (1, 7, 100, 100000):
            for strategy, k in [(0, 0), (1, 0), (2, 0), (2, 1), (2, 3), (2, 6), (2, 7)]:
                for mtpb in (1024, 512):
                    st, ng, cpb = plan(species, strategy, k, cells, mtpb)
                    want_ng = of.orc().orc_group_count(strategy, cells, species, mtpb, k)
                    ocpb = C.c_double()
                    ost = of.orc().orc_plan_cells_per_block(strategy, cells, species, mtpb, k, C.byref(ocpb))
                    assert st == ost, (species, cells, strategy, k, mtpb)
                    if st == 0:
                        assert ng == want_ng and cpb == ocpb.value


def test_plan_errors():
    assert plan(156, 2, 7, 10)[0] == -2  # InvalidGrouping
    assert plan(2000, 2, 1, 10)[0] == -3  # UnsupportedMechanism
    assert plan(156, 2, 1, 0)[0] == -1  # no cells
    assert plan(156, 9, 1, 10)[0] == -1  # unknown strategy


def export_schedule(rp, ci, k, with_t):
    species = len(rp) - 1
    info = np.zeros(12, np.int32)
    lib = _native.b200()
    rp = np.ascontiguousarray(rp, np.int32)
    ci = np.ascontiguousarray(ci, np.int32)
    st = lib.bc_schedule_export(species, of.ptr(rp), of.ptr(ci), k, with_t, of.ptr(info), None, None, None, None,
                                None, None)
    assert st == 0
    n, P, Q, W, R, RV, S, St, xs, txs, cost, tcost = info.tolist()
    nnz = int(rp[-1])
    words = np.zeros(max(S * W * 32, 1), np.uint32)
    vpos = np.zeros(k * nnz, np.int32)
    twords = np.zeros(max(St * W * 32, 1), np.uint32)
    tvpos = np.zeros(k * nnz, np.int32)
    xpos = np.zeros(n, np.int32)
    txpos = np.zeros(n, np.int32)
    st = lib.bc_schedule_export(species, of.ptr(rp), of.ptr(ci), k, with_t, of.ptr(info), of.ptr(words),
                                of.ptr(vpos), of.ptr(xpos), of.ptr(twords), of.ptr(tvpos), of.ptr(txpos))
    assert st == 0
    return dict(n=n, P=P, Q=Q, W=W, R=R, RV=RV, S=S, St=St, words=words, vpos=vpos, twords=twords, tvpos=tvpos,
                xpos=xpos, txpos=txpos, xslots=xs, txslots=txs, cost=cost, tcost=tcost)


def emulate_pass(words, vpos, vals, S, LW, x, n, xpos, xslots):
    """team_spmv() of bc_block.cuh in exact double arithmetic: publish x at its
    slots, then every lane walks its schedule."""
    V = np.zeros(S * LW)
    V[vpos] = vals
    X = np.full(xslots, np.nan)  # unused slots must never be read
    X[xpos] = x
    x = X
    y = np.zeros(n)
    for L in range(LW):
        acc = 0.0
        for t in range(S):
            e = int(words[t * LW + L])
            acc = acc + float(V[t * LW + L]) * float(x[e & 0xFFF])
            if e >> 31:
                y[(e >> 12) & 0xFFF] = acc
                acc = 0.0
    return y


def ref_spmv(rp, ci, vals, x, k, s, nnz):
    y = np.zeros(k * s)
    for c in range(k):
        for i in range(s):
            acc = 0.0
            for e in range(rp[i], rp[i + 1]):
                acc = acc + float(vals[c * nnz + e]) * float(x[c * s + ci[e]])
            y[c * s + i] = acc
    return y


def ref_spmv_t(rp, ci, vals, x, k, s, nnz):
    y = np.zeros(k * s)
    for c in range(k):
        for i in range(s):
            for e in range(rp[i], rp[i + 1]):
                j = c * s + ci[e]
                y[j] = y[j] + float(vals[c * nnz + e]) * float(x[c * s + i])
    return y


@pytest.mark.parametrize("species,k,density,seed", [(9, 1, 0.4, 0), (40, 3, 0.2, 1), (156, 1, 0.0, 2),
                                                    (100, 5, 0.05, 3), (17, 30, 0.3, 4)])
def test_schedule_reproduces_spmv_order(species, k, density, seed):
    rng = np.random.default_rng(seed)
    if density == 0.0:
        m = Mechanism(156, 468, 0)
        rp, ci = m.row_ptr, m.col_idx
    else:
        rp, ci, _, _ = random_batch(rng, 1, species, density)
    nnz = int(rp[-1])
    sc = export_schedule(rp, ci, k, 1)
    LW = sc["W"] * 32
    vals = rng.uniform(-1, 1, k * nnz) * 10.0 ** rng.integers(-8, 8, k * nnz)
    x = rng.uniform(-1, 1, k * species)
    y = emulate_pass(sc["words"], sc["vpos"], vals, sc["S"], LW, x, k * species, sc["xpos"], sc["xslots"])
    np.testing.assert_array_equal(of.bits(y), of.bits(ref_spmv(rp, ci, vals, x, k, species, nnz)))
    yt = emulate_pass(sc["twords"], sc["tvpos"], vals, sc["St"], LW, x, k * species, sc["txpos"], sc["txslots"])
    np.testing.assert_array_equal(of.bits(yt), of.bits(ref_spmv_t(rp, ci, vals, x, k, species, nnz)))
    assert sc["S"] * LW >= k * nnz  # every value has a slot
    assert sorted(sc["vpos"].tolist()) == sorted(set(sc["vpos"].tolist()))
    assert len(set(sc["xpos"].tolist())) == k * species and sc["xpos"].max() < sc["xslots"]


def emulate_team_reduce(vals, n, P, W, R):
    """team_reduce() of bc_block.cuh: per-lane tree over R slots, cross-warp
    tree over W, xor butterfly over 32 lanes (lane 0's value)."""
    lanes = {}
    for w in range(W):
        for lane in range(32):
            t = [0.0] * R
            for j in range(R):
                i = (j * W + w) * 32 + lane
                t[j] = float(vals[i]) if i < n else 0.0
            s = R // 2
            while s >= 1:
                for j in range(s):
                    t[j] = t[j] + t[j + s]
                s //= 2
            lanes[(w, lane)] = t[0]
    part = []
    for lane in range(32):
        u = [lanes[(w, lane)] for w in range(W)]
        s = W // 2
        while s >= 1:
            for q in range(s):
                u[q] = u[q] + u[q + s]
            s //= 2
        part.append(u[0])
    if P >= 32:
        masks = [16, 8, 4, 2, 1]
    else:
        masks = []
        m = P // 2
        while m >= 1:
            masks.append(m)
            m //= 2
    for mask in masks:
        part = [part[l] + part[l ^ mask] for l in range(32)]
    return part[0]


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 17, 31, 32, 33, 100, 156, 255, 256, 257, 312, 500, 936, 1024, 1500,
                               2048])
def test_reduction_geometry_reproduces_tree(n):
    info = np.zeros(12, np.int32)
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.arange(n, dtype=np.int32)
    assert _native.b200().bc_schedule_export(n, of.ptr(rp), of.ptr(ci), 1, 0, of.ptr(info), None, None, None,
                                              None, None, None) == 0
    _, P, Q, W, R, RV = info.tolist()[:6]
    assert W * R == Q and P >= n
    rng = np.random.default_rng(n)
    for _ in range(5):
        v = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 12, n)
        v[rng.random(n) < 0.1] = -0.0
        slots = np.zeros(P)
        slots[:n] = v
        want = of.orc().orc_tree_reduce_in_place(of.ptr(slots), P)
        got = emulate_team_reduce(v, n, P, W, R)
        assert of.bits(got) == of.bits(want)


def export_tmem_schedule(rp, ci, k, pair=0, team=1):
    species = len(rp) - 1
    rp = np.ascontiguousarray(rp, np.int32)
    ci = np.ascontiguousarray(ci, np.int32)
    info = np.zeros(9, np.int32)
    lib = _native.b200()
    assert lib.bc_tmem_schedule_export(species, of.ptr(rp), of.ptr(ci), k, pair, team, of.ptr(info), None, None,
                                       None, None) == 0
    S, copies = int(info[0]), int(info[5])
    mult = 2 if pair else 1
    words = np.zeros(S * 32 * team, np.uint16)
    vidx = np.zeros(S * 32 * team, np.int32)
    xpos = np.zeros(copies * k * species * mult, np.int32)
    yslot = np.zeros(k * species * mult, np.int32)
    assert lib.bc_tmem_schedule_export(species, of.ptr(rp), of.ptr(ci), k, pair, team, of.ptr(info), of.ptr(words),
                                       of.ptr(vidx), of.ptr(xpos), of.ptr(yslot)) == 0
    return dict(S=S, xslots=int(info[1]), zero_slot=int(info[2]), yslots=int(info[3]), cost=int(info[4]),
                copies=copies, model=int(info[6]), streams=int(info[7]), ystream=int(info[8]), team=team, words=words,
                vidx=vidx, xpos=xpos.reshape(copies, -1), yslot=yslot)


def emulate_tmem_spmv(sc, vals, x):
    """tmem_spmv() of bc_tmem.cuh in exact double arithmetic: zero-initialised
    X|Y, publish x, lanes walk 16-bit words (byte offset; bit 15 of step
    4c+2's word flags a row ending on step 4c+3, bit 15 of step 4c's a row
    ending on step 4c+1 with one stream or 4c+2 with two), stream s of lane
    L runs on steps s mod streams; its k-th row -> Y[s*ystream + k*32 + L]."""
    S, ST, LW = sc["S"], sc["streams"], 32 * sc["team"]
    X = np.zeros(sc["xslots"] + 1)
    for xp in sc["xpos"]:  # every copy of the gather vector
        X[xp] = x
    Y = np.zeros(sc["yslots"] + LW)
    words = sc["words"].reshape(S, LW)
    for L in range(LW):
        acc, k = [0.0] * ST, [0] * ST
        for t in range(S):
            w = int(words[t, L])
            vi = int(sc["vidx"][t * LW + L])
            a = float(vals[vi]) if vi >= 0 else 0.0
            s = t % ST
            acc[s] = acc[s] + a * float(X[(w & 0x7FFF) // 8])
            if (t & 1) and (w & 0x8000):
                raise AssertionError("end flag on an odd step")
            flag = t - 1 if (t & 3) == 3 else (t & ~3 if (t & 3) == ST else -1)
            if flag >= 0 and int(words[flag, L]) & 0x8000:
                Y[s * sc["ystream"] + k[s] * LW + L] = acc[s]
                k[s] += 1
                acc[s] = 0.0
    return Y[sc["yslot"]]


@pytest.mark.parametrize("pair,team", [(0, 1), (1, 1), (0, 2), (1, 2), (0, 4)])
@pytest.mark.parametrize("species,k,density,seed", [(9, 1, 0.4, 0), (40, 3, 0.2, 1), (156, 1, 0.0, 2),
                                                    (100, 2, 0.05, 3), (17, 15, 0.3, 4), (60, 1, 0.02, 5)])
def test_tmem_schedule_reproduces_spmv_order(species, k, density, seed, pair, team):
    rng = np.random.default_rng(seed)
    if density == 0.0:
        m = Mechanism(156, 468, 0)
        rp, ci = m.row_ptr, m.col_idx
    else:
        rp, ci, _, _ = random_batch(rng, 1, species, density)
        if seed == 5:  # empty rows
            rp = rp.copy()
            keep = np.ones(len(ci), bool)
            for r in (3, 7):
                keep[rp[r]:rp[r + 1]] = False
            lens = np.diff(rp) * 1
            lens[[3, 7]] = 0
            ci = ci[keep]
            rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nnz = int(rp[-1])
    sc = export_tmem_schedule(rp, ci, k, pair, team)
    assert sc["S"] % 4 == 0
    vals = rng.uniform(-1, 1, k * nnz) * 10.0 ** rng.integers(-8, 8, k * nnz)
    n = k * species
    x = rng.uniform(-1, 1, n * (2 if pair else 1))
    x[rng.random(len(x)) < 0.05] = np.inf  # padding must never touch x (0*inf = NaN)
    y = emulate_tmem_spmv(sc, vals, x)
    with np.errstate(invalid="ignore"):
        np.testing.assert_array_equal(of.bits(y[:n]), of.bits(ref_spmv(rp, ci, vals, x[:n], k, species, nnz)))
        if pair:  # BiCG's A^T p~ in the same pass, ascending source rows (csr.cpp:129-142)
            np.testing.assert_array_equal(of.bits(y[n:]), of.bits(ref_spmv_t(rp, ci, vals, x[n:], k, species, nnz)))
    used = sc["vidx"][sc["vidx"] >= 0]
    assert sorted(used.tolist()) == sorted(list(range(k * nnz)) * (2 if pair else 1))


@pytest.mark.parametrize("species,k", [(156, 6), (100, 8), (60, 17)])
def test_tmem_schedule_coupled_team4_two_streams(species, k):
    """Four-warp teams on coupled groups above 512 rows (Block-cells(N): 936 at
    M156) run two row streams per lane: the walk still reproduces spmv's
    per-row order (csr.cpp:90-101) bit for bit."""
    rng = np.random.default_rng(species + k)
    if species == 156:
        m = Mechanism(156, 468, 0)
        rp, ci = m.row_ptr, m.col_idx
    else:
        rp, ci, _, _ = random_batch(rng, 1, species, 0.1)
    nnz = int(rp[-1])
    sc = export_tmem_schedule(rp, ci, k, 0, 4)
    assert sc["streams"] == 2 and sc["S"] % 4 == 0
    vals = rng.uniform(-1, 1, k * nnz) * 10.0 ** rng.integers(-8, 8, k * nnz)
    n = k * species
    x = rng.uniform(-1, 1, n)
    y = emulate_tmem_spmv(sc, vals, x)
    np.testing.assert_array_equal(of.bits(y[:n]), of.bits(ref_spmv(rp, ci, vals, x, k, species, nnz)))


# --- latency-mode schedule (bc_latency_plan.cpp) ------------------------------

def export_latency_schedule(rp, ci, k, bicg, threads):
    lib = _native.b200()
    _p = of.ptr
    rp = np.ascontiguousarray(rp, np.int32)
    ci = np.ascontiguousarray(ci, np.int32)
    species = len(rp) - 1
    info = np.zeros(8, np.int32)
    assert lib.bc_latency_schedule_export(species, _p(rp), _p(ci), k, bicg, threads, _p(info), *([None] * 7)) == 0
    n, P, T, lmax, L, xslots, model, ok = (int(v) for v in info)
    out = dict(n=n, P=P, T=T, lmax=lmax, L=L, xslots=xslots, model=model, ok=ok)
    if not ok:
        return out
    rowof, steps, didx = np.zeros(T, np.int32), np.zeros(T, np.int32), np.zeros(P, np.int32)  # noqa: E501
    rvi, tvi = np.zeros(L * T, np.int32), np.zeros(L * T, np.int32)
    rxo, txo = np.zeros(L * T, np.uint16), np.zeros(L * T, np.uint16)
    assert lib.bc_latency_schedule_export(species, _p(rp), _p(ci), k, bicg, threads, _p(info), _p(rowof), _p(steps),
                                          _p(rvi), _p(rxo), _p(tvi), _p(txo), _p(didx)) == 0
    out.update(rowof=rowof, steps=steps, didx=didx, rvi=rvi.reshape(L, T), rxo=rxo.reshape(L, T),
               tvi=tvi.reshape(L, T), txo=txo.reshape(L, T))
    return out


def emulate_latency_spmv(sc, vals, x, xt=None):
    """The latency kernel's SpMV as it runs: every thread its row in its
    warp's private gather region (x at slot = row, 16 zero slots, p~ after
    them), entries in table order from +0.0 up to its warp's step count;
    the sums land in Y[row]."""
    P, T = sc["P"], sc["T"]
    X = np.zeros(sc["xslots"])
    X[:len(x)] = x
    if xt is not None:
        X[P + 16:P + 16 + len(xt)] = xt
    Y, YT = np.zeros(P), np.zeros(P)
    for t in range(T):
        row = sc["rowof"][t]
        if row < 0:
            continue
        for tab_v, tab_o, out in ((sc["rvi"], sc["rxo"], Y), (sc["tvi"], sc["txo"], YT if xt is not None else None)):
            if out is None:
                continue
            acc = 0.0
            for e in range(sc["steps"][t]):
                vi = tab_v[e, t]
                a = vals[vi] if vi >= 0 else 0.0
                with np.errstate(invalid="ignore"):
                    acc = acc + a * X[tab_o[e, t] // 8]
            out[row] = acc
    return Y, YT


@pytest.mark.parametrize("bicg", [0, 1])
@pytest.mark.parametrize("species,k,density,seed", [(156, 1, 0.0, 0), (40, 3, 0.2, 1), (70, 2, 0.1, 2),
                                                    (33, 1, 0.3, 3), (100, 2, 0.05, 4)])
def test_latency_schedule_reproduces_spmv_order(species, k, density, seed, bicg):
    """Every row (and, for BiCG, A^T row) in CSR / ascending-source-row order
    from +0.0 with padding that only adds +0.0: bit-identical to csr.cpp's
    spmv / spmv_transpose; each value used exactly once per pass; rows dealt
    longest first with per-warp step counts covering every row."""
    rng = np.random.default_rng(seed)
    if density == 0.0:
        m = Mechanism(156, 468, 0)
        rp, ci = m.row_ptr, m.col_idx
    else:
        rp, ci, _, _ = random_batch(rng, 1, species, density)
    nnz = int(rp[-1])
    n = k * species
    threads = 32 * ((n + 31) // 32)
    sc = export_latency_schedule(rp, ci, k, bicg, threads)
    assert sc["ok"] and sc["T"] == threads
    assert sorted(int(r) for r in sc["rowof"] if r >= 0) == list(range(n))
    lens = np.diff(rp)
    for t in range(threads):
        r = sc["rowof"][t]
        if r >= 0:
            assert sc["steps"][t] >= lens[r % species]
    vals = rng.uniform(-1, 1, k * nnz) * 10.0 ** rng.integers(-8, 8, k * nnz)
    x = rng.uniform(-1, 1, n)
    xt = rng.uniform(-1, 1, n) if bicg else None
    Y, YT = emulate_latency_spmv(sc, vals, x, xt)
    np.testing.assert_array_equal(of.bits(Y[:n]), of.bits(ref_spmv(rp, ci, vals, x, k, species, nnz)))
    if bicg:
        np.testing.assert_array_equal(of.bits(YT[:n]), of.bits(ref_spmv_t(rp, ci, vals, xt, k, species, nnz)))
    used = sc["rvi"][sc["rvi"] >= 0]
    assert sorted(used.tolist()) == list(range(k * nnz))
    # padding gathers one of the 16 zero slots
    pad = sc["rxo"][sc["rvi"] < 0] // 8
    assert ((pad >= sc["P"]) & (pad < sc["P"] + 16)).all()
