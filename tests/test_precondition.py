"""Preconditioner, phase 1 of the pipeline (precondition.cpp:37-153), SURVEY.md §8(f)
row 3.  The device path reproduces the reference's operation order, so every
result is checked BITWISE against the unmodified reference (oracle/_ref).  The
reference-side hooks are test infrastructure (oracle/ref_harness.cpp)."""
import os
import sys

import numpy as np
import pytest

import paper_2602_06694_b200 as nq

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
import oracle as O  # noqa: E402

pytestmark = pytest.mark.skipif(not O.reference_available(), reason="reference library not built")


def ref():
    return O.reference()


def stats(rng, cols, batches=3, rows=37):
    ss, cnt, tau = np.zeros(cols), 0, 0.0
    for b in range(batches):
        x = rng.standard_normal((rows + b, cols)) * np.linspace(0.1, 3.0, cols)
        ss, cnt, tau = ref().accumulate_stats(ss, cnt, tau, x, 0.9)
    return ss, cnt, tau


@pytest.mark.parametrize("with_out", [False, True])
@pytest.mark.parametrize("gamma", [0.0, 0.25, 1.0])
def test_build_preconditioner_bitwise(with_out, gamma):
    rng = np.random.default_rng(3)
    ins = stats(rng, 50)
    outs = stats(rng, 30) if with_out else None
    want = ref().build_preconditioner(*ins, *(outs if outs else (None, 0, 0.0)), gamma, 1e-6)
    got = nq.build_preconditioner(nq.ChannelStats(*ins),
                                  nq.ChannelStats(*outs) if outs else None, gamma, 1e-6)
    assert np.array_equal(got.diag_in, want[0])
    if with_out:
        assert np.array_equal(got.diag_out, want[1])
    else:
        assert got.diag_out.size == 0
    assert got.tau_max == want[2]


def test_build_preconditioner_errors():
    ins = nq.ChannelStats(np.ones(4), 0, 1.0)
    with pytest.raises(nq.EmptyStats):
        nq.build_preconditioner(ins, None, 0.1, 1e-6)
    ins.sample_count = 3
    with pytest.raises(nq.EmptyStats):
        nq.build_preconditioner(ins, nq.ChannelStats(np.ones(2), 0, 0.0), 0.1, 1e-6)
    with pytest.raises(nq.Error):
        nq.build_preconditioner(ins, None, 1.5, 1e-6)
    with pytest.raises(nq.Error):
        nq.build_preconditioner(ins, None, 0.5, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("cols", [1, 7, 256, 1000])
def test_accumulate_stats_bitwise(cols):
    rng = np.random.default_rng(cols)
    got = nq.ChannelStats.zeros(cols)
    ss, cnt, tau = np.zeros(cols), 0, 0.0
    for b, rows in enumerate([17, 1, 64, 0, 33]):
        x = rng.standard_normal((rows, cols)) * rng.uniform(0.01, 5.0, cols)
        nq.accumulate_stats(got, x, 0.95)
        if rows:
            ss, cnt, tau = ref().accumulate_stats(ss, cnt, tau, x, 0.95)
    assert np.array_equal(got.sum_squares, ss)
    assert got.sample_count == cnt and got.tau == tau


@pytest.mark.gpu
def test_accumulate_stats_device_tensor_and_errors():
    import torch
    rng = np.random.default_rng(9)
    x = rng.standard_normal((40, 24))
    a, b = nq.ChannelStats.zeros(24), nq.ChannelStats.zeros(24)
    nq.accumulate_stats(a, x, 0.5)
    nq.accumulate_stats(b, torch.from_numpy(x).cuda(), 0.5)
    assert np.array_equal(a.sum_squares, b.sum_squares) and a.tau == b.tau
    bad = x.copy()
    bad[3, 5] = np.nan
    with pytest.raises(nq.NonFiniteInput):
        nq.accumulate_stats(nq.ChannelStats.zeros(24), bad, 0.5)
    with pytest.raises(nq.Error):
        nq.accumulate_stats(nq.ChannelStats.zeros(24), x, 1.0)
    with pytest.raises(nq.DimensionMismatch):
        nq.accumulate_stats(nq.ChannelStats.zeros(23), x, 0.5)


@pytest.mark.gpu
@pytest.mark.parametrize("diags", ["both", "in", "out", "none"])
def test_precondition_and_unprecondition_bitwise(diags):
    rng = np.random.default_rng(11)
    w = rng.standard_normal((70, 45))
    dout = rng.uniform(0.2, 3.0, 70) if diags in ("both", "out") else None
    din = rng.uniform(0.2, 3.0, 45) if diags in ("both", "in") else None
    p = nq.Preconditioner(din if din is not None else np.empty(0),
                          dout if dout is not None else np.empty(0))
    assert np.array_equal(nq.precondition_weight(w, p), ref().precondition_weight(w, dout, din))
    f = rng.standard_normal((70, 12))
    d = dout if dout is not None else np.empty(0)
    want = ref().unprecondition_rows(f, dout) if dout is not None else f
    assert np.array_equal(nq.unprecondition_rows(f, d), want)
