"""Pins the CPU oracle (oracle/nq_oracle.c) before anything is compared to it.

1. The reference's own known-answer vectors (test_packed.cpp, test_linalg.cpp,
   test_admm.cpp, test_balance.cpp, test_storage.cpp) on the restatement.
2. Bitwise equality of the restatement with the unmodified reference library
   (oracle/_ref, compiled from /root/reference) on seeded random inputs.
3. Bitwise equality with the committed golden fixtures (tests/golden/).
4. A subset of the reference's property tests, run on the restatement.
"""
import glob
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, bits_of, rel


# --------------------------------------------------------------------------
# 1. known-answer vectors
# --------------------------------------------------------------------------
def test_kat_binarize_sign_of_zero(chk):  # test_packed.cpp:39-54
    b = chk.binarize(np.array([[0.3, -0.2], [0.0, -5.0]]))
    assert b.tolist() == [[1, -1], [1, -1]]
    assert chk.binarize(np.array([[-0.0]]))[0, 0] == 1.0  # x < 0, not signbit
    with pytest.raises(O.OracleError) as e:
        chk.binarize(np.array([[np.nan]]))
    assert e.value.code == 2


def test_kat_pack(chk):  # test_packed.cpp:56-72
    assert chk.pack_signs(np.array([[1, -1, 1, -1.0]])).tolist() == [[5]]
    assert chk.pack_signs(np.ones((1, 33))).tolist() == [[0xFFFFFFFF, 1]]
    assert chk.pack_signs(-np.ones((1, 32))).tolist() == [[0]]
    with pytest.raises(O.OracleError) as e:
        chk.pack_signs(np.full((1, 3), 0.5))
    assert e.value.code == 3


def test_kat_unpack(chk):  # test_packed.cpp:74-84
    assert chk.unpack_signs(np.array([[5]], np.uint32), 1, 4).tolist() == [[1, -1, 1, -1]]
    with pytest.raises(O.OracleError) as e:
        chk.unpack_signs(np.array([[5 | (1 << 10)]], np.uint32), 1, 4)
    assert e.value.code == 4


def test_kat_reconstruct_and_gemv(chk):  # test_packed.cpp:94-141
    ones = chk.make_factorized_layer(np.ones((3, 1)), np.ones((4, 1)), [1, 1, 1], [1, 1, 1, 1])
    assert np.all(chk.reconstruct_dense(ones) == 1.0)
    cancel = chk.make_factorized_layer(np.ones((1, 2)), np.array([[1.0, -1.0]]), [1.0], [1.0])
    assert chk.reconstruct_dense(cancel)[0, 0] == 0.0
    ones5 = chk.make_factorized_layer(np.ones((3, 1)), np.ones((5, 1)), [1] * 3, [1] * 5)
    x = chk.rng(74).gaussian(5)
    assert np.allclose(chk.gemv_packed(ones5, x), x.sum(), rtol=1e-12)
    assert np.all(chk.gemv_packed(ones5, np.zeros(5)) == 0.0)
    with pytest.raises(O.OracleError) as e:
        chk.gemv_packed(ones5, np.zeros(4))
    assert e.value.code == 1


def test_kat_rank_rule(chk):  # test_storage.cpp:230-237
    assert chk.rank_for_target_bpw(64, 64, 1.0) == 16
    assert chk.rank_for_target_bpw(4096, 4096, 1.0) == 2032
    assert chk.rank_for_target_bpw(4096, 4096, 0.55) == 1110
    assert chk.rank_for_target_bpw(2000, 2000, 0.01) == 1
    with pytest.raises(O.OracleError) as e:
        chk.rank_for_target_bpw(4096, 4096, 1e-4)
    assert e.value.code == 8
    # SURVEY.md §8 rank table (verified there against the reference)
    for (n, m), rs in {(4096, 4096): (2032, 1622, 1110), (11008, 4096): (2969, 2372, 1626),
                       (5120, 5120): (2544, 2032, 1392), (13824, 5120): (3720, 2973, 2039),
                       (8192, 8192): (4080, 3261, 2237), (28672, 8192): (6356, 5081, 3488)
                       }.items():
        assert tuple(chk.rank_for_target_bpw(n, m, t) for t in (1.0, 0.8, 0.55)) == rs


def test_kat_linalg(chk):  # test_linalg.cpp:26-93
    x = chk.cholesky_solve(np.array([[4.0, 2], [2, 3]]), np.array([[1.0], [0.0]]))
    assert np.allclose(x[:, 0], [0.375, -0.25], rtol=1e-12)
    b = np.arange(1, 7, dtype=float).reshape(3, 2)
    assert np.array_equal(chk.cholesky_solve(np.eye(3), b), b)
    with pytest.raises(O.OracleError) as e:
        chk.cholesky_solve(np.array([[1.0, 5], [2, 1]]), np.zeros((2, 1)))
    assert e.value.code == 7
    with pytest.raises(O.OracleError) as e:
        chk.cholesky_solve(np.array([[1.0, 0], [0, -5]]), np.zeros((2, 1)))
    assert e.value.code == 33
    s, left, right, _ = chk.top_singular_pair(np.full((2, 2), 2.0), 200, 1e-12)
    assert abs(s - 4.0) <= 4e-10
    assert np.allclose(left, 2 ** -0.5, rtol=1e-9) and np.allclose(right, 2 ** -0.5, rtol=1e-9)
    s, left, right, _ = chk.top_singular_pair(np.array([[3.0, 0], [0, 1]]), 500, 1e-13)
    assert abs(s - 3.0) <= 3e-8 and abs(abs(left[0]) - 1) <= 1e-6


def test_kat_svid_and_balance(chk):  # test_admm.cpp:50-56, test_balance.cpp:26-36
    p = np.array([[2.0, -2], [-2, 2]])
    assert rel(chk.svid(p), p) <= 1e-10
    c = np.full((3, 5), 2.5)
    assert rel(chk.svid(c), c) <= 1e-10
    lu, lv, s1, s2, eta = chk.balance_and_extract_scales(np.array([[2.0]]), np.array([[8.0]]))
    assert np.isclose(eta, 2.0) and np.isclose(lu[0, 0], 4.0) and np.isclose(lv[0, 0], 4.0)
    assert np.isclose(s1[0], 4.0) and np.isclose(s2[0], 4.0)


# --------------------------------------------------------------------------
# 2. restatement == reference, bitwise
# --------------------------------------------------------------------------
def test_rng_and_half_bitwise(chk, ref):
    for seed in (0, 1, 0xB1A5E001, 2 ** 63 + 5):
        a, b = chk.rng(seed), ref.rng(seed)
        assert np.array_equal(a.u64(100), b.u64(100))
        assert np.array_equal(a.gaussian(1000), b.gaussian(1000))
        assert np.array_equal(a.uniform(0.25, 2.0, 100), b.uniform(0.25, 2.0, 100))
        assert np.array_equal(a.sign(100), b.sign(100))
        assert np.array_equal(a.index(37, 100), b.index(37, 100))
    all_halves = np.arange(65536, dtype=np.uint16)
    da, db = chk.half_to_double(all_halves), ref.half_to_double(all_halves)
    assert np.array_equal(np.isnan(da), np.isnan(db))
    ok = ~np.isnan(da)
    assert np.array_equal(da[ok], db[ok])
    x = np.concatenate([chk.rng(9).gaussian(20000) * 10.0 ** np.arange(-8, 8).repeat(1250),
                        da[ok], [0.0, -0.0, 65504.0, 65520.0, 1e9, 5.96e-8, 2.98e-8, 2.99e-8]])
    assert np.array_equal(chk.double_to_half(x), ref.double_to_half(x))


def test_forward_bitwise(chk, ref):
    rng = chk.rng(75)
    for trial in range(12):
        n, m, r = (int(v) for v in 1 + rng.index(300, 3))
        lay = O.synthetic_layer(chk, 100 + trial, n, m, r)
        x = chk.rng(200 + trial).gaussian(m)
        assert np.array_equal(chk.gemv_packed(lay, x), ref.gemv_packed(lay, x))
        assert np.array_equal(chk.gemv_packed_f32(lay, x), ref.gemv_packed_f32(lay, x))
        assert np.array_equal(chk.reconstruct_dense(lay), ref.reconstruct_dense(lay))
        X = chk.rng(300 + trial).matrix(m, 1 + trial)
        assert np.array_equal(chk.gemm_packed(lay, X), ref.gemm_packed(lay, X))
        s = np.where(chk.rng(400 + trial).gaussian(n * r).reshape(n, r) < 0, -1.0, 1.0)
        assert np.array_equal(chk.pack_signs(s), ref.pack_signs(s))


def test_linalg_admm_bitwise(chk, ref):
    rng = chk.rng(5)
    for trial in range(6):
        n, m = 3 + int(rng.index(40)), 3 + int(rng.index(40))
        r = 1 + int(rng.index(min(n, m)))
        w = O.synthetic_weight(chk, 50 + trial, n, m)
        for x, y in zip(chk.top_singular_pair(w, 1000, 1e-13), ref.top_singular_pair(w, 1000, 1e-13)):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        assert chk.spectral_norm_estimate(w) == ref.spectral_norm_estimate(w)
        assert np.array_equal(chk.svid(w), ref.svid(w))
        ua, va = chk.truncated_svd_factors(w, r)
        ub, vb = ref.truncated_svd_factors(w, r)
        assert np.array_equal(ua, ub) and np.array_equal(va, vb)
        fixed = chk.rng(60 + trial).matrix(m, r)
        z = chk.rng(70 + trial).matrix(n, r)
        l = chk.rng(80 + trial).matrix(n, r)
        assert np.array_equal(chk.admm_factor_solve(w, fixed, z, l, 0.7, 1e-3),
                              ref.admm_factor_solve(w, fixed, z, l, 0.7, 1e-3))
        cfg = O.AdmmConfig.make(rank=r, max_iters=60)
        for x, y in zip(chk.admm_factorize(w, cfg)[:3], ref.admm_factorize(w, cfg)[:3]):
            assert np.array_equal(x, y)
        la, ea, _, _ = chk.factorize_layer(w, cfg)
        lb, eb, _, _ = ref.factorize_layer(w, cfg)
        assert ea == eb and np.array_equal(la.u, lb.u) and np.array_equal(la.v, lb.v)
        assert np.array_equal(la.s1, lb.s1) and np.array_equal(la.s2, lb.s2)


# --------------------------------------------------------------------------
# 3. committed fixtures (made from the reference by tests/golden/make_golden.py)
# --------------------------------------------------------------------------
SMALL_FIXTURES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "admm_*.npz"))
                        if int(np.load(p)["n"]) * int(np.load(p)["m"]) <= 160 * 128)


@pytest.mark.parametrize("path", SMALL_FIXTURES, ids=os.path.basename)
def test_restatement_matches_golden(chk, path):
    g = np.load(path)
    w = O.synthetic_weight(chk, int(g["seed"]), int(g["n"]), int(g["m"]))
    cfg = O.AdmmConfig.make(rank=int(g["r"]), max_iters=int(g["max_iters"]))
    lay, err, trace, res = chk.factorize_layer(w, cfg)
    assert err == float(g["rel_err"])
    assert np.array_equal(lay.u, g["u"]) and np.array_equal(lay.v, g["v"])
    assert np.array_equal(lay.s1, g["s1"]) and np.array_equal(lay.s2, g["s2"])
    assert res["iteration"] == int(g["iteration"])
    assert np.array_equal(trace, g["trace"])


def test_golden_fixture_set_present():
    names = {os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "admm_*.npz"))}
    assert {"admm_w64x48_b1.0.npz", "admm_w128_b1.0.npz", "admm_w256_b1.0.npz"} <= names


# --------------------------------------------------------------------------
# 4. reference property tests, on the restatement
# --------------------------------------------------------------------------
def test_gemv_vs_dense_and_gemm_vs_gemv(chk):  # test_packed.cpp:143-217
    rng = chk.rng(75)
    for trial in range(20):
        n, m = 1 + int(rng.index(200)), 1 + int(rng.index(200))
        r = 1 + int(rng.index(64))
        lay = O.synthetic_layer(chk, 1000 + trial, n, m, r)
        x = chk.rng(2000 + trial).gaussian(m)
        dense = chk.reconstruct_dense(lay)
        y = chk.gemv_packed(lay, x)
        assert np.linalg.norm(dense @ x - y) <= 1e-10 * (1 + np.linalg.norm(dense @ x))
        X = chk.rng(3000 + trial).matrix(m, 5)
        Y = chk.gemm_packed(lay, X)
        for c in range(5):
            assert np.array_equal(Y[:, c], chk.gemv_packed(lay, X[:, c]))


def test_admm_monotone_descent(chk):  # test_admm.cpp:222-235
    w = chk.rng(29).matrix(16, 12)
    cfg = O.AdmmConfig.make(rank=2, max_iters=120, rho_start=16 * chk.spectral_norm_estimate(w),
                            rho_end=16 * chk.spectral_norm_estimate(w))
    trace = chk.admm_factorize(w, cfg)[2]
    assert len(trace) >= 2
    assert np.all(trace[1:] <= trace[:-1] + 1e-8 * (1 + np.abs(trace[:-1])))


def test_admm_in_class_rank1(chk):  # test_admm.cpp:185-203 (subset of the 100 seeds)
    rng = chk.rng(27)
    hits = 0
    for _ in range(20):
        n, m = 2 + int(rng.index(63)), 2 + int(rng.index(63))
        a = rng.sign(n) * rng.uniform(0.5, 2.0, n)
        b = rng.sign(m) * rng.uniform(0.5, 2.0, m)
        w = np.outer(a, b)
        _, err, _, _ = chk.factorize_layer(w, O.AdmmConfig.make(rank=1))
        hits += err <= 1e-3
    assert hits >= 19


def test_sign_agreement_helper():
    w = np.array([[0b1011, 0xFFFFFFFF]], np.uint32)
    b = bits_of(w, 36)
    assert b[0, :4].tolist() == [True, True, False, True] and b[0, 32:].all()
