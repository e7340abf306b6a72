"""GPU parity of the persistent decode-pass kernel (decode_pass.cu) through the C ABI.

A pass runs many decode steps in one launch.  Its per-layer arithmetic is the
per-call kernel's (decode.cu): with an external input both compute the
activation bound from max|x|, and a chained step takes it from the producer's
published max|y| (= max|x| of its input), so every output is held BITWISE
equal to the per-call kernel on the same input, and within the north-star bar
of the reference's gemv_packed_f32 (packed.cpp:201-204).
"""
import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-3
TIGHT_TOL = 2e-5


def rand_layer(nq, rng, n, m, r, ctx=None):
    k = (r + 31) // 32
    u = rng.integers(0, 2 ** 32, size=(n, k), dtype=np.uint32)
    v = rng.integers(0, 2 ** 32, size=(m, k), dtype=np.uint32)
    if r % 32:
        mask = np.uint32((1 << (r % 32)) - 1)
        u[:, -1] &= mask
        v[:, -1] &= mask
    # scales ~ 1/sqrt(r), 1/sqrt(m): keeps chained fp16 activations O(1)
    s1 = (rng.uniform(0.25, 2.0, n) / np.sqrt(r)).astype(np.float16).view(np.uint16)
    s2 = (rng.uniform(0.25, 2.0, m) / np.sqrt(m)).astype(np.float16).view(np.uint16)
    lay = nq.DeviceLayer.upload_f16(n, m, r, u, v, s1, s2, ctx)
    return lay, O.Layer(n, m, r, u, v, s1.view(np.float16).astype(np.float64),
                        s2.view(np.float16).astype(np.float64))


def per_call(unit, x, ys, nq):
    if isinstance(unit, nq.DecodeGroup):
        unit.gemv_device(x, ys)
    else:
        unit.gemv_device(x, ys[0])


def block_model(nq, rng, dims, dtype, chained):
    """One Llama-like block repeated: qkv group, o, gate/up group, down.
    dims = (d, f, r_att, r_mlp).  Chained: o reads q's output, gate/up read
    o's output, down reads gate's output, the next block reads down's output."""
    import torch
    d, f, ra, rm = dims
    q, hq = rand_layer(nq, rng, d, d, ra)
    k, hk = rand_layer(nq, rng, d // 4, d, ra // 4 + 3)
    v, hv = rand_layer(nq, rng, d // 4, d, ra // 4 + 3)
    o, ho = rand_layer(nq, rng, d, d, ra)
    g, hg = rand_layer(nq, rng, f, d, rm)
    u, hu = rand_layer(nq, rng, f, d, rm)
    dn, hd = rand_layer(nq, rng, d, f, rm)
    qkv = nq.DecodeGroup([q, k, v])
    gu = nq.DecodeGroup([g, u])
    new = lambda n: torch.empty(n, device="cuda", dtype=dtype)  # noqa: E731
    x0 = torch.randn(d, device="cuda", dtype=dtype)
    yq, yk, yv, yo, yg, yu, yd = new(d), new(d // 4), new(d // 4), new(d), new(f), new(f), new(d)
    if chained:
        xo, xg, xd = yq, yo, yg
    else:
        xo, xg, xd = (torch.randn(d, device="cuda", dtype=dtype),
                      torch.randn(d, device="cuda", dtype=dtype),
                      torch.randn(f, device="cuda", dtype=dtype))
    steps = [(qkv, x0, [yq, yk, yv]), (o, xo, [yo]), (gu, xg, [yg, yu]), (dn, xd, [yd])]
    host = {id(qkv): [hq, hk, hv], id(o): [ho], id(gu): [hg, hu], id(dn): [hd]}
    keep = [q, k, v, o, g, u, dn]
    return steps, host, keep


def run_and_check(nq, chk, steps, host, oracle_check=True):
    """Launch the pass, then re-run every step with the per-call kernel on the
    inputs the pass actually saw: bitwise equality, and the oracle bar."""
    import torch
    p = nq.DecodePass(steps)
    p.launch()
    torch.cuda.synchronize()
    outs = [[y.clone() for y in ys] for _, _, ys in steps]
    ins = [x.clone() for _, x, _ in steps]
    # per-call reference on a snapshot of each step's input
    for (unit, _, ys), x, got in zip(steps, ins, outs):
        ref = [torch.empty_like(y) for y in ys]
        per_call(unit, x, ref, nq)
        torch.cuda.synchronize()
        for a, b in zip(got, ref):
            assert torch.equal(a, b), "pass output differs from the per-call kernel"
        if oracle_check:
            xs = x.float().cpu().numpy()
            for hl, a in zip(host[id(unit)], got):
                assert rel(a.float().cpu().numpy(), chk.gemv_packed_f32(hl, xs)) <= FWD_TOL
    return p, outs


@pytest.mark.parametrize("chained", [False, True], ids=["independent", "chained"])
def test_pass_bitwise_equals_per_call(nq, chk, chained):
    import torch
    rng = np.random.default_rng(11 + chained)
    steps, host, keep = [], {}, []
    for blk in range(3):
        s, h, kp = block_model(nq, rng, (1024, 2752, 400, 600), torch.float16, chained)
        if chained and steps:  # the next block reads the previous block's down output
            s[0] = (s[0][0], steps[-1][2][0], s[0][2])
        steps += s
        host.update(h)
        keep += kp
    p, outs = run_and_check(nq, chk, steps, host)
    # replays: the kernel clears its own accumulators -> identical bits
    for _ in range(3):
        p.launch()
        torch.cuda.synchronize()
        for (_, _, ys), want in zip(steps, outs):
            for y, w in zip(ys, want):
                assert torch.equal(y, w)


def test_pass_tails_and_fp32(nq, chk):
    import torch
    rng = np.random.default_rng(5)
    shapes = [(300, 320, 320), (77, 100, 45), (2048, 512, 511), (1, 3000, 1), (64, 28672, 40),
              (513, 257, 193), (1, 1, 1)]
    steps, host = [], {}
    for n, m, r in shapes:
        lay, h = rand_layer(nq, rng, n, m, r)
        x = torch.randn(m, device="cuda", dtype=torch.float32)
        steps.append((lay, x, [torch.empty(n, device="cuda", dtype=torch.float32)]))
        host[id(lay)] = [h]
    _, outs = run_and_check(nq, chk, steps, host)
    for (lay, x, _), got in zip(steps, outs):
        want = chk.gemv_packed_f32(host[id(lay)][0], x.cpu().numpy())
        assert rel(got[0].cpu().numpy(), want) <= TIGHT_TOL


@pytest.mark.parametrize("env", [
    {"NQB_PASS_SPLIT": "1"},
    {"NQB_PASS_SPLIT": "2", "NQB_PASS_ITEM_SLABS": "1"},
    {"NQB_PASS_SPLIT": "8", "NQB_PASS_ITEM_SLABS": "3", "NQB_PASS_WAVE_DIV": "2",
     "NQB_PASS_WAVE_DIV2": "2", "NQB_PASS_MIN_RINGS_KB": "0"},
    {"NQB_PASS_PLAN_SLABS": "2", "NQB_PASS_RING1_PCT": "50", "NQB_PASS_WARPS1": "6"},
])
def test_pass_work_split_is_bitwise_invariant(nq, chk, env, monkeypatch):
    """Outputs do not depend on the SM partitions, the pass plans, the work items or
    the ring waves (small rings wrap and reuse slots many times)."""
    import torch
    rng = np.random.default_rng(21)
    steps, host, keep = block_model(nq, rng, (2048, 5504, 900, 1300), torch.float16, False)
    _, a = run_and_check(nq, chk, steps, host)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, b = run_and_check(nq, chk, steps, host, oracle_check=False)
    for x, y in zip(a, b):
        for u, v in zip(x, y):
            assert torch.equal(u, v)


def test_pass_70b_gate_up_group_and_down(nq, chk):
    """A 32 MB gate/up group streams through the ring in many chunks."""
    import torch
    rng = np.random.default_rng(70)
    g, hg = rand_layer(nq, rng, 28672, 8192, 3488)
    u, hu = rand_layer(nq, rng, 28672, 8192, 3488)
    dn, hd = rand_layer(nq, rng, 8192, 28672, 3488)
    gu = nq.DecodeGroup([g, u])
    x = torch.randn(8192, device="cuda", dtype=torch.float16)
    yg, yu = (torch.empty(28672, device="cuda", dtype=torch.float16) for _ in range(2))
    yd = torch.empty(8192, device="cuda", dtype=torch.float16)
    steps = [(gu, x, [yg, yu]), (dn, yg, [yd])]
    run_and_check(nq, chk, steps, {id(gu): [hg, hu], id(dn): [hd]})


def test_pass_in_cuda_graph(nq, chk):
    import torch
    ctx = nq.context(0)
    rng = np.random.default_rng(3)
    steps, host, keep = block_model(nq, rng, (1024, 2752, 400, 600), torch.float16, True)
    p, outs = run_and_check(nq, chk, steps, host, oracle_check=False)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.bind_torch_stream()
        with ctx.capture() as cap:
            p.launch()
        for _ in range(3):
            for _, _, ys in steps:
                for y in ys:
                    y.zero_()
            # the chained inputs are outputs: restore x0 only (it is external)
            cap.graph.launch()
            torch.cuda.synchronize()
            for (_, _, ys), want in zip(steps, outs):
                for y, w in zip(ys, want):
                    assert torch.equal(y, w)
    torch.cuda.synchronize()
    ctx.bind_torch_stream()


def test_pass_non_finite_input_propagates_nan(nq, chk):
    import torch
    rng = np.random.default_rng(9)
    a, _ = rand_layer(nq, rng, 300, 400, 64)
    b, _ = rand_layer(nq, rng, 200, 300, 64)
    x = torch.randn(400, device="cuda", dtype=torch.float16)
    x[7] = float("nan")
    ya = torch.empty(300, device="cuda", dtype=torch.float16)
    yb = torch.empty(200, device="cuda", dtype=torch.float16)
    p = nq.DecodePass([(a, x, [ya]), (b, ya, [yb])])
    p.launch()
    torch.cuda.synchronize()
    assert torch.isnan(ya).all() and torch.isnan(yb).all()
    x[7] = float("inf")
    p.launch()
    torch.cuda.synchronize()
    assert torch.isnan(ya).all() and torch.isnan(yb).all()
    x[7] = 0.5  # recovers on the next launch (flags live in the cleared arena)
    p.launch()
    torch.cuda.synchronize()
    assert torch.isfinite(ya).all() and torch.isfinite(yb).all()


def test_pass_rejects_bad_steps(nq):
    import torch
    rng = np.random.default_rng(4)
    a, _ = rand_layer(nq, rng, 64, 64, 16)
    x = torch.randn(64, device="cuda", dtype=torch.float16)
    with pytest.raises(nq.DimensionMismatch):
        nq.DecodePass([(a, x, [torch.empty(63, device="cuda", dtype=torch.float16)])])
    with pytest.raises(nq.Error):  # output aliases its own input
        nq.DecodePass([(a, x, [x])])


def test_pass_run_host_registered_and_pageable_agree(nq, chk):
    """nqb_pass_run_host with registered (nqb_host_register), plain pinned and
    pageable host buffers gives the device pass's outputs bit for bit."""
    import torch
    rng = np.random.default_rng(33)
    steps, host, keep = block_model(nq, rng, (1024, 2752, 400, 600), torch.float16, False)
    p = nq.DecodePass(steps)
    p.launch()
    torch.cuda.synchronize()
    want = [y.cpu().numpy().copy() for _, _, ys in steps for y in ys]
    ctx = p.ctx
    for mode in ("pageable", "pinned", "registered"):
        if mode == "pageable":
            hx = [x.cpu().numpy().copy() for _, x, _ in steps]
            hy = [np.empty_like(w) for w in want]
        else:
            hx = [x.cpu().pin_memory().numpy() for _, x, _ in steps]
            hy = [torch.empty(w.shape, dtype=torch.float16).pin_memory().numpy() for w in want]
        if mode == "registered":
            for a in hx + hy:
                ctx.register_host(a)
        p.run_host(hx, hy)
        for a, b in zip(hy, want):
            assert np.array_equal(a.view(np.uint16), b.view(np.uint16)), mode
        if mode == "registered":
            for a in hx + hy:
                ctx.unregister_host(a)
    p.free()


def test_pass_host_io_bound_buffers(nq, chk):
    """nqb_pass_io_*: pinned and registered host buffers bound once give the device
    pass's outputs bit for bit on every run; pageable buffers are refused."""
    import torch
    rng = np.random.default_rng(34)
    steps, host, keep = block_model(nq, rng, (1024, 2752, 400, 600), torch.float16, False)
    p = nq.DecodePass(steps)
    p.launch()
    torch.cuda.synchronize()
    want = [y.cpu().numpy().copy() for _, _, ys in steps for y in ys]
    ctx = p.ctx
    hx = [x.cpu().pin_memory().numpy() for _, x, _ in steps]
    hy = [torch.empty(w.shape, dtype=torch.float16).pin_memory().numpy() for w in want]
    io = p.host_io(hx, hy)
    for _ in range(3):
        for a in hy:
            a[...] = 0
        io.run()
        for a, b in zip(hy, want):
            assert np.array_equal(a.view(np.uint16), b.view(np.uint16))
    io.close()
    hxr = [x.cpu().numpy().copy() for _, x, _ in steps]  # pageable, then registered
    with pytest.raises(nq.Error):
        p.host_io(hxr, hy)
    for a in hxr:
        ctx.register_host(a)
    io = p.host_io(hxr, hy)
    io.run()
    for a, b in zip(hy, want):
        assert np.array_equal(a.view(np.uint16), b.view(np.uint16))
    io.close()
    for a in hxr:
        ctx.unregister_host(a)
    p.free()
