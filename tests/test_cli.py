"""nqb_cli: the reference CLI's infer / verify / bench (nanoquant_main.cpp:147-159,
:253-340) on the GPU over the C ABI, with the reference's exit codes (0 / 2 / 3)."""
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_06694_b200 as nq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_06694_b200", "nqb_cli")
GOLD = os.path.join(ROOT, "tests", "golden", "nqpk_small.nqpk")
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


def write_nqmx(path, a):
    a = np.asarray(a, np.float32)
    with open(path, "wb") as f:
        f.write(b"NQMX" + struct.pack("<III", 1, a.shape[0], a.shape[1]) + a.tobytes())


def read_nqmx(path):
    b = open(path, "rb").read()
    assert b[:4] == b"NQMX"
    _, rows, cols = struct.unpack_from("<III", b, 4)
    return np.frombuffer(b, np.float32, rows * cols, 16).reshape(rows, cols)


def test_cli_usage_and_validation_exit_codes():
    assert os.path.exists(CLI), "build() makes paper_2602_06694_b200/nqb_cli"
    assert run("--help").returncode == 0
    assert run().returncode == 2
    assert run("frobnicate", "--model", GOLD).returncode == 2
    assert run("verify").returncode == 2  # missing --model


@pytest.mark.gpu
def test_cli_verify_reference_written_model():
    r = run("verify", "--model", GOLD)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 3 and all("words=ok gemv=ok" in l for l in lines), r.stdout


@pytest.mark.gpu
def test_cli_infer_chain_matches_reference_gemm(tmp_path):
    import oracle as O
    chk = O.restated()
    dims = [(48, 64, 20), (80, 48, 33), (33, 80, 17)]  # x(64) -> 48 -> 80 -> 33
    layers = [O.synthetic_layer(chk, 0xD00D + i, n, m, r) for i, (n, m, r) in enumerate(dims)]
    model = tmp_path / "chain.nqpk"
    nq.write_packed_model(str(model), [(f"l{i}", nq.FactorizedLayer(l.n, l.m, l.r, l.u, l.v, l.s1, l.s2))
                                       for i, l in enumerate(layers)])
    x = chk.rng(0xFEED).gaussian(64 * 3).reshape(64, 3).astype(np.float32)
    xin, yout = tmp_path / "x.nqmx", tmp_path / "y.nqmx"
    write_nqmx(xin, x)
    r = run("infer", "--model", str(model), "--vector-in", str(xin), "--out", str(yout), "--batch")
    assert r.returncode == 0, r.stderr
    got = read_nqmx(yout).astype(np.float64)
    want = x.astype(np.float64)
    for l in layers:  # the file holds binary16 scales: the reference sees the snapped ones
        ls = O.Layer(l.n, l.m, l.r, l.u, l.v, chk.snap_half(l.s1), chk.snap_half(l.s2))
        want = chk.gemm_packed(ls, want)
    assert got.shape == want.shape
    assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)
    # a single column is required without --batch (nanoquant_main.cpp:150-152)
    assert run("infer", "--model", str(model), "--vector-in", str(xin), "--out",
               str(yout)).returncode == 2


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    out = tmp_path / "bench.csv"
    r = run("bench", "--model", GOLD, "--iters", "20", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = out.read_text().strip().splitlines()
    assert rows[0].startswith("layer,n,m,r,decode_us") and len(rows) == 4
