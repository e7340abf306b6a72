"""GPU parity of the fused decode kernel (decode.cu) through the C ABI.

The kernel quantises activations to 38-bit fixed point and accumulates
exactly in integers, so besides the north-star bar (1e-3 relative to the
reference's gemv_packed_f32, packed.cpp:201-204) it is held to a much tighter
internal bar, and to bitwise identity wherever the arithmetic must agree:
grouped vs single-layer launches, PDL on/off, graph replay vs direct calls.
"""
import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-3    # north_star
TIGHT_TOL = 2e-5  # what the 38-bit fixed point actually delivers


def to_nq(nq, lay):
    return nq.FactorizedLayer(lay.n, lay.m, lay.r, lay.u, lay.v, lay.s1, lay.s2)


def dev_layer(nq, chk, seed, n, m, r):
    lay = O.synthetic_layer(chk, seed, n, m, r)
    return lay, nq.DeviceLayer.upload(to_nq(nq, lay))


# K tails of every kind: r % 256 in {0, 64, 128, 192, ragged}, m likewise
TAIL_SHAPES = [(300, 320, 320), (200, 448, 130), (77, 100, 45), (40, 1000, 500),
               (513, 257, 193), (16, 64, 64), (17, 65, 65), (1, 3000, 1),
               (2048, 512, 511), (64, 28672, 40), (1, 1, 1), (2, 33, 2)]


@pytest.mark.parametrize("shape", TAIL_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_decode_tails_vs_reference(nq, chk, shape):
    n, m, r = shape
    lay, dev = dev_layer(nq, chk, 0xD0 + n * 7 + m, n, m, r)
    x = chk.rng(n + 3 * m).gaussian(m).astype(np.float32)
    want = chk.gemv_packed_f32(lay, x)
    got = dev.gemv_f32(x)
    assert rel(got, want) <= TIGHT_TOL


@pytest.mark.parametrize("name,n,m,r", [("l7_q", 4096, 4096, 1622), ("l70_gate", 28672, 8192, 3488),
                                        ("l70_down", 8192, 28672, 3488)])
def test_decode_tight_on_target_shapes(nq, chk, name, n, m, r):
    lay, dev = dev_layer(nq, chk, 0xB1A5E100 + n + m, n, m, r)
    x = chk.rng(0xB1A5E002).gaussian(m).astype(np.float32)
    assert rel(dev.gemv_f32(x), chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL


def test_decode_zero_and_wide_dynamic_range(nq, chk):
    n, m, r = 500, 700, 96
    lay, dev = dev_layer(nq, chk, 91, n, m, r)
    assert np.all(dev.gemv_f32(np.zeros(m, np.float32)) == 0)
    x = chk.rng(92).gaussian(m).astype(np.float32)
    x[17] = 3.0e4  # one outlier: the fixed point is set by the bound, the rest still count
    x[18] = -1e-30
    want = chk.gemv_packed_f32(lay, x)
    assert rel(dev.gemv_f32(x), want) <= FWD_TOL


def test_group_bitwise_equals_single_layers(nq, chk):
    import torch
    m = 4096
    specs = [(4096, 1622), (1024, 300), (4096, 1622)]  # q, (short) k, v
    lays, devs = [], []
    for i, (n, r) in enumerate(specs):
        lay, dev = dev_layer(nq, chk, 0x6000 + i, n, m, r)
        lays.append(lay)
        devs.append(dev)
    grp = nq.DecodeGroup(devs)
    x = torch.from_numpy(chk.rng(5).gaussian(m).astype(np.float16)).cuda()
    ys = [torch.empty(n, dtype=torch.float16, device="cuda") for n, _ in specs]
    grp.gemv_device(x, ys)
    singles = []
    for d, (n, _) in zip(devs, specs):
        y = torch.empty(n, dtype=torch.float16, device="cuda")
        d.gemv_device(x, y)
        singles.append(y)
    torch.cuda.synchronize()
    for lay, y, s in zip(lays, ys, singles):
        assert torch.equal(y, s)
        want = chk.gemv_packed_f32(lay, x.float().cpu().numpy())
        assert rel(y.float().cpu().numpy(), want) <= FWD_TOL
    assert grp.stream_bytes >= sum(r * (n + m) // 8 for n, r in specs)


def test_interleaved_layers_share_scratch(nq, chk):
    """Different plans back to back on one stream (t-buffer reuse, dirty rows)."""
    import torch
    shapes = [(8192, 8192, 2237), (64, 300, 17), (4096, 11008, 2372), (1000, 8192, 45)]
    items = []
    for i, (n, m, r) in enumerate(shapes):
        lay, dev = dev_layer(nq, chk, 0x7000 + i, n, m, r)
        x = chk.rng(0x7100 + i).gaussian(m).astype(np.float32)
        items.append((lay, dev, x, chk.gemv_packed_f32(lay, x)))
    xs = [torch.from_numpy(x).cuda() for _, _, x, _ in items]
    ys = [torch.empty(lay.n, dtype=torch.float32, device="cuda") for lay, _, _, _ in items]
    first = None
    for rep in range(3):
        for (lay, dev, _, _), xd, yd in zip(items, xs, ys):
            dev.gemv_device(xd, yd)
        torch.cuda.synchronize()
        outs = [y.cpu().numpy().copy() for y in ys]
        for (_, _, _, want), got in zip(items, outs):
            assert rel(got, want) <= TIGHT_TOL
        if first is None:
            first = outs
        else:
            for a, b in zip(first, outs):
                assert np.array_equal(a, b)


def test_pdl_off_and_graph_replay_bitwise(nq, chk):
    import torch
    ctx = nq.context(0)
    lay_a, a = dev_layer(nq, chk, 0x8001, 4096, 4096, 1622)
    lay_b, b = dev_layer(nq, chk, 0x8002, 11008, 4096, 2372)
    # fp32 chain (b's fp16 output would overflow: |y_b| ~ 1e7)
    xa = torch.from_numpy(chk.rng(1).gaussian(4096).astype(np.float32)).cuda()
    ya = torch.empty(4096, dtype=torch.float32, device="cuda")
    yb = torch.empty(11008, dtype=torch.float32, device="cuda")

    def run():
        a.gemv_device(xa, ya)
        b.gemv_device(ya[:4096], yb)  # b reads a's output: a real dependency
        torch.cuda.synchronize()
        return ya.clone(), yb.clone()

    ref_a, ref_b = run()
    want_b = chk.gemv_packed_f32(lay_b, ref_a.cpu().numpy())
    assert rel(ref_b.cpu().numpy(), want_b) <= TIGHT_TOL
    ctx.set_pdl(False)
    try:
        pa, pb = run()
    finally:
        ctx.set_pdl(True)
    assert torch.equal(pa, ref_a) and torch.equal(pb, ref_b)
    side = torch.cuda.Stream()  # graphs cannot capture the legacy NULL stream
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.bind_torch_stream()
        with ctx.capture() as cap:
            a.gemv_device(xa, ya)
            b.gemv_device(ya[:4096], yb)
        for _ in range(3):
            ya.zero_()
            yb.zero_()
            cap.graph.launch()
            torch.cuda.synchronize()
            assert torch.equal(ya, ref_a) and torch.equal(yb, ref_b)
    torch.cuda.synchronize()
    ctx.bind_torch_stream()


def test_host_dropin_pinned_and_pageable_agree(nq, chk):
    """nqb_gemv_f32_host writes a pinned y in place over the host link and a
    pageable y through a device copy: same bits either way."""
    import torch
    lay, dev = dev_layer(nq, chk, 0x5EED, 700, 900, 300)
    x = chk.rng(77).gaussian(900).astype(np.float32)
    pageable = dev.gemv_f32(x)
    pinned = torch.empty(700, dtype=torch.float32).pin_memory().numpy()
    dev.gemv_f32(x, out=pinned)
    xp = torch.from_numpy(x.copy()).pin_memory().numpy()
    pinned2 = torch.empty(700, dtype=torch.float32).pin_memory().numpy()
    dev.gemv_f32(xp, out=pinned2)
    assert np.array_equal(pageable, pinned) and np.array_equal(pageable, pinned2)
    assert rel(pageable, chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL


@pytest.mark.parametrize("shape", [(300, 320, 320), (77, 100, 45), (2048, 512, 511), (4096, 4096, 1622),
                                   (1, 1, 1)], ids=lambda s: "x".join(map(str, s)))
def test_compact_and_pipelined_instances_bitwise(nq, chk, shape, monkeypatch):
    """The two kernel instances (compact loop, software-pipelined slab runs;
    NQB_DEC_BIG_KB picks per plan) do the same integer arithmetic: bitwise equal."""
    n, m, r = shape
    lay = O.synthetic_layer(chk, 0xB16 + n + m, n, m, r)
    x = chk.rng(5 * n + m).gaussian(m).astype(np.float32)
    out = {}
    for kb in ("0", "1000000"):
        monkeypatch.setenv("NQB_DEC_BIG_KB", kb)
        out[kb] = nq.DeviceLayer.upload(to_nq(nq, lay)).gemv_f32(x)
    assert np.array_equal(out["0"], out["1000000"])
    assert rel(out["0"], chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL


# ---- activation range, non-finite inputs, ring mode -------------
@pytest.mark.parametrize("scale", [1e-4, 1e-2, 1.0, 1e2, "heavy"])
def test_fp16_decode_across_activation_scales(nq, chk, scale):
    """The activation exponent comes from the device max|x| for binary16 inputs
    too, so tiny and large activations keep full relative precision."""
    import torch
    lays, devs = [], []
    for i, (n, r) in enumerate([(4096, 1622), (1024, 300)]):
        lay, dev = dev_layer(nq, chk, 0x5C00 + i, n, 4096, r)
        lays.append(lay)
        devs.append(dev)
    rng = np.random.default_rng(17)
    if scale == "heavy":
        x = rng.standard_t(1.5, 4096) * 0.05
        x = np.clip(x, -6e4, 6e4)
    else:
        x = rng.standard_normal(4096) * scale
    xh = torch.from_numpy(x.astype(np.float16)).cuda()
    xs = xh.float().cpu().numpy()
    y = torch.empty(4096, dtype=torch.float16, device="cuda")
    devs[0].gemv_device(xh, y)
    want = chk.gemv_packed_f32(lays[0], xs)
    ok = np.isfinite(want).all() and np.abs(want).max() < 6e4
    if ok:
        assert rel(y.float().cpu().numpy(), want) <= FWD_TOL
    grp = nq.DecodeGroup(devs)
    ys = [torch.empty(l.n, dtype=torch.float16, device="cuda") for l in lays]
    grp.gemv_device(xh, ys)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], y)
    for lay, yy in zip(lays, ys):
        want = chk.gemv_packed_f32(lay, xs)
        if np.isfinite(want).all() and np.abs(want).max() < 6e4:
            assert rel(yy.float().cpu().numpy(), want) <= FWD_TOL


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_non_finite_input_gives_nan_outputs(nq, chk, bad, dtype):
    """gemv_two_stage propagates a NaN/Inf activation into every output
    (t_k = +-Inf for all k, then y_i = sum of mixed-sign Infs = NaN); the
    kernel flags the input in its max|x| pass and writes NaN."""
    import torch
    lay, dev = dev_layer(nq, chk, 0xBAD, 300, 400, 96)
    x = chk.rng(3).gaussian(400).astype(np.float32)
    x[123] = bad
    want = chk.gemv_packed_f32(lay, x)
    assert np.isnan(want).all()
    if dtype == "f32":
        got = dev.gemv_f32(x)
    else:
        xd = torch.from_numpy(x.astype(np.float16)).cuda()
        yd = torch.empty(300, dtype=torch.float16, device="cuda")
        dev.gemv_device(xd, yd)
        got = yd.float().cpu().numpy()
    assert np.isnan(got).all()


@pytest.mark.parametrize("kb", ["24", "48"])
def test_forced_ring_mode(nq, chk, kb, monkeypatch):
    """A small stream buffer forces ring mode (sections streamed through slots)."""
    import torch
    monkeypatch.setenv("NQB_DEC_SMEM_KB", kb)
    lays, devs = [], []
    for i, (n, m, r) in enumerate([(4096, 4096, 1622), (2048, 4096, 900)]):
        lay, dev = dev_layer(nq, chk, 0x41A0 + i, n, m, r)
        lays.append(lay)
        devs.append(dev)
    x = chk.rng(8).gaussian(4096).astype(np.float32)
    for lay, dev in zip(lays, devs):
        assert rel(dev.gemv_f32(x), chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL
    grp = nq.DecodeGroup(devs)
    xd = torch.from_numpy(x).cuda()
    ys = [torch.empty(l.n, dtype=torch.float32, device="cuda") for l in lays]
    grp.gemv_device(xd, ys)
    torch.cuda.synchronize()
    for lay, y in zip(lays, ys):
        assert rel(y.cpu().numpy(), chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL


def test_70b_gate_up_group_and_high_bitrate_layer(nq, chk):
    """Streams larger than the buffer (ring mode by default): a 70B gate/up group
    and a 70B q layer at 1.0 bit (r = 4080)."""
    import torch
    rng = np.random.default_rng(99)
    specs = [(28672, 8192, 3488), (28672, 8192, 3488)]
    devs, lays = [], []
    for i, (n, m, r) in enumerate(specs):
        lay, dev = dev_layer(nq, chk, 0x70A0 + i, n, m, r)
        lays.append(lay)
        devs.append(dev)
    grp = nq.DecodeGroup(devs)
    x = chk.rng(12).gaussian(8192).astype(np.float32)
    ys = [torch.empty(n, dtype=torch.float32, device="cuda") for n, _, _ in specs]
    grp.gemv_device(torch.from_numpy(x).cuda(), ys)
    torch.cuda.synchronize()
    for lay, y in zip(lays, ys):
        assert rel(y.cpu().numpy(), chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL
    lay, dev = dev_layer(nq, chk, 0x70B0, 8192, 8192, 4080)
    x = chk.rng(13).gaussian(8192).astype(np.float32)
    assert rel(dev.gemv_f32(x), chk.gemv_packed_f32(lay, x)) <= TIGHT_TOL


def test_graph_then_bigger_upload_keeps_graph_valid(nq, chk):
    """A graph captured before an upload that grows the decode state keeps
    replaying correctly (old state retired, not freed)."""
    import torch
    ctx = nq.context(0)
    lay, dev = dev_layer(nq, chk, 0x6A1, 512, 512, 128)
    x = torch.from_numpy(chk.rng(1).gaussian(512).astype(np.float32)).cuda()
    y = torch.empty(512, dtype=torch.float32, device="cuda")
    dev.gemv_device(x, y)
    torch.cuda.synchronize()
    want = y.clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.bind_torch_stream()
        with ctx.capture() as cap:
            dev.gemv_device(x, y)
    torch.cuda.synchronize()
    ctx.bind_torch_stream()
    # a group far larger than the current state capacity (rows of t)
    big = [dev_layer(nq, chk, 0x6B0 + i, 64, 512, 16000)[1] for i in range(3)]
    grp = nq.DecodeGroup(big)
    with torch.cuda.stream(side):
        for _ in range(3):
            y.zero_()
            cap.graph.launch()
            torch.cuda.synchronize()
            assert torch.equal(y, want)
    torch.cuda.synchronize()
    ctx.bind_torch_stream()
    del grp


def test_decode_co_resident_under_busy_stream_and_two_contexts(nq, chk):
    """The per-call kernel's grid barrier needs every CTA resident: the launch is
    cooperative, so decode completes correctly while another stream keeps the
    SMs busy, and while a second context (own stream) decodes concurrently."""
    import threading

    import torch
    n, m, r = 4096, 4096, 1622
    lay = O.synthetic_layer(chk, 0xC0, n, m, r)
    x = chk.rng(0xC1).gaussian(m).astype(np.float32)
    want = chk.gemv_packed_f32(lay, x)
    fl = nq.FactorizedLayer(n, m, r, lay.u, lay.v, lay.s1, lay.s2)
    ctx2 = nq.Context(0)
    d1 = nq.DeviceLayer.upload(fl, nq.context(0))
    d2 = nq.DeviceLayer.upload(fl, ctx2)
    busy = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda")
    with torch.cuda.stream(busy):
        for _ in range(40):
            a = torch.tanh(a @ a)  # keeps every SM occupied for a while
    outs = {}

    def run(dev, key):
        outs[key] = [dev.gemv_f32(x) for _ in range(20)]

    th = threading.Thread(target=run, args=(d2, "b"))
    th.start()
    run(d1, "a")
    th.join(timeout=120)
    torch.cuda.synchronize()
    for key in ("a", "b"):
        assert len(outs[key]) == 20
        for y in outs[key]:
            assert rel(y, want) <= 2e-5
    ctx2.close()
