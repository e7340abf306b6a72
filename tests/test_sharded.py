"""Layer-sharded ADMM initialisation driver: plan, payload format and the
world-size-2 gather over gloo (CPU).  The per-matrix work is a deterministic
stand-in here (the device factorisation is covered by test_gpu_admm.py and
the GPU test below); what is tested is the sharding and the collective."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_06694_b200 import sharded as S


def fake_factorize(spec, index):
    """Deterministic stand-in for device_factorize (same payload shapes)."""
    r = max(1, min(spec.n, spec.m) // 3)
    rng = np.random.default_rng(spec.seed)
    k = (r + 31) // 32
    u = rng.integers(0, 2 ** 32, size=(spec.n, k), dtype=np.uint32)
    v = rng.integers(0, 2 ** 32, size=(spec.m, k), dtype=np.uint32)
    if r % 32:
        u[:, -1] &= np.uint32((1 << (r % 32)) - 1)
        v[:, -1] &= np.uint32((1 << (r % 32)) - 1)
    s1 = rng.uniform(0.25, 2, spec.n).astype(np.float16).view(np.uint16)
    s2 = rng.uniform(0.25, 2, spec.m).astype(np.float16).view(np.uint16)
    return S.PackedMatrix(index, spec.n, spec.m, r, u, v, s1, s2, 0.5 + index * 1e-3, 40 + index,
                          True, 0.01)


def small_specs():
    shapes = [(64, 48), (96, 160), (128, 128), (40, 300), (200, 64), (33, 77), (64, 64)]
    return [S.MatrixSpec(f"m{i}", n, m, 1000 + i) for i, (n, m) in enumerate(shapes * 3)]


def test_llama2_7b_specs_and_ranks():
    specs = S.llama2_7b_specs()
    assert len(specs) == 224
    assert sum(1 for s in specs if (s.n, s.m) == (4096, 4096)) == 128
    assert S.rank_for(4096, 4096, 1.0) == 2032 and S.rank_for(11008, 4096, 1.0) == 2969
    assert S.rank_for(4096, 4096, 0.55) == 1110  # test_storage.cpp:230-237


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lpt_assignment_is_a_balanced_partition(world):
    specs = S.llama2_7b_specs()
    a = S.lpt_assign(specs, world, 1.0)
    flat = sorted(i for lst in a for i in lst)
    assert flat == list(range(len(specs)))
    loads = [sum(S.cost(specs[i], 1.0) for i in lst) for lst in a]
    assert max(loads) / (sum(loads) / world) < 1.02  # 7B classes split evenly
    assert a == S.lpt_assign(specs, world, 1.0)       # deterministic


def test_payload_roundtrip_bitwise():
    items = [fake_factorize(s, i) for i, s in enumerate(small_specs()[:5])]
    back = S.unpack_shard(S.pack_shard(items))
    assert len(back) == len(items)
    for a, b in zip(items, back):
        assert (a.index, a.n, a.m, a.r, a.iterations, a.converged) == \
            (b.index, b.n, b.m, b.r, b.iterations, b.converged)
        for f in ("u", "v", "s1", "s2"):
            assert np.array_equal(getattr(a, f), getattr(b, f))
        assert a.rel_error == b.rel_error


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rep = S.sharded_init(small_specs(), 1.0, factorize=fake_factorize)
        if rank == 0:
            out.put({i: (p.u.tobytes(), p.v.tobytes(), p.s1.tobytes(), p.s2.tobytes(), p.r)
                     for i, p in rep.matrices.items()})
        else:
            assert rep is None
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_equals_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = S.sharded_init(small_specs(), 1.0, factorize=fake_factorize)  # world 1
    assert sorted(got) == sorted(want.matrices)
    for i, pm in want.matrices.items():
        assert got[i] == (pm.u.tobytes(), pm.v.tobytes(), pm.s1.tobytes(), pm.s2.tobytes(), pm.r)


@pytest.mark.gpu
def test_device_factorize_small_matrix_matches_layer_path():
    """The product work function on a 64x48 matrix: packed words round-trip and
    the metrics are those of nqb_factorize_layer."""
    spec = S.MatrixSpec("w", 64, 48, 12345)
    pm = S.device_factorize(spec, 0, 1.0)
    assert pm.r == 11 and pm.u.shape == (64, 1) and pm.v.shape == (48, 1)  # storage.cpp:124-141
    assert 0 < pm.rel_error < 1.5 and pm.iterations >= 1
    rt = S.unpack_shard(S.pack_shard([pm]))[0]
    assert np.array_equal(rt.u, pm.u) and np.array_equal(rt.s2, pm.s2)


def _device_worker(rank, world, port, out):
    """One rank of a real multi-rank run: the device factorisation (libnqb on
    cuda:0, both ranks share the GPU) + the gloo gather of packed factors."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rep = S.sharded_init(device_specs(), 1.0)
        if rank == 0:
            out.put({i: (p.u.tobytes(), p.v.tobytes(), p.s1.tobytes(), p.s2.tobytes(), p.r,
                         p.rel_error, p.iterations) for i, p in rep.matrices.items()})
        else:
            assert rep is None
    finally:
        dist.destroy_process_group()


def device_specs():
    """Four small matrices, W from the reference Rng (SURVEY §8(d) row 4 seeds)."""
    shapes = [(64, 48), (96, 160), (128, 128), (200, 64)]
    return [S.MatrixSpec(f"d{i}", n, m, 0x7B000000 + i) for i, (n, m) in enumerate(shapes)]


@pytest.mark.gpu
def test_device_sharded_world2_gather_bitwise_equals_world1():
    """SURVEY §8(d) protocol: the gathered packed factors of a 2-rank device run
    equal a single-rank run bit for bit (same matrices, same metrics)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = S.sharded_init(device_specs(), 1.0)
    assert sorted(got) == sorted(want.matrices) == [0, 1, 2, 3]
    for i, pm in want.matrices.items():
        assert got[i] == (pm.u.tobytes(), pm.v.tobytes(), pm.s1.tobytes(), pm.s2.tobytes(), pm.r,
                          pm.rel_error, pm.iterations)
        assert pm.svd_power_iters > 0 and pm.seconds_svd > 0


def test_synthetic_weight_matches_reference_rng():
    """The product's W generator (libnqb host code) is the reference Rng stream:
    bitwise equal to rng.hpp via oracle/_ref, including the fp32 snap."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import oracle as O
    from paper_2602_06694_b200 import nanoquant as nq
    chk = O.reference() if O.reference_available() else O.restated()
    for seed, n, m in [(0x7B000000, 3, 5), (0x7B000000 + 7 * 3 + 4, 257, 300),
                       (0xB1A5E001, 64, 4096)]:
        w = nq.synthetic_weight(seed, n, m)
        ref = O.synthetic_weight(chk, seed, n, m)
        assert np.array_equal(w.view(np.uint64), ref.view(np.uint64))
    spec = S.MatrixSpec("b3.up", 64, 96, 0x7B000000 + 7 * 3 + 5)
    assert np.array_equal(S.synthetic_weight(spec), O.synthetic_weight(chk, spec.seed, 64, 96))
