"""NQPK packed-model files (io.hpp:27-54, io.cpp:139-193), SURVEY.md §8(f) row 1.

* Parsing a file written by the reference serializer (tests/golden/nqpk_small.*,
  made by tests/golden/make_nqpk.py).
* Byte-exact serialisation, with the ParseError / IoError cases of
  deserialize_packed_model / read_file.
* GPU tests: the file goes straight to the device layout and decodes like the
  reference, and device layers are written back byte for byte.
"""
import os
import struct

import numpy as np
import pytest

import paper_2602_06694_b200 as nq

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "nqpk_small.nqpk")


def golden():
    z = np.load(os.path.join(HERE, "golden", "nqpk_small.npz"))
    out = []
    for i, name in enumerate(z["names"]):
        n, m, r = (int(x) for x in z[f"dims{i}"])
        out.append((str(name), n, m, r, z[f"u{i}"], z[f"v{i}"], z[f"s1h{i}"], z[f"s2h{i}"]))
    return out


def test_reads_reference_written_file():
    layers = nq.read_packed_model(GOLD)
    want = golden()
    assert [nm for nm, _ in layers] == [w[0] for w in want]
    for (name, lay), (_, n, m, r, u, v, s1h, s2h) in zip(layers, want):
        assert (lay.n, lay.m, lay.r) == (n, m, r)
        assert np.array_equal(lay.u, u) and np.array_equal(lay.v, v)
        # binary16 scales widen exactly
        assert np.array_equal(lay.s1.astype(np.float16).view(np.uint16), s1h)
        assert np.array_equal(lay.s2.astype(np.float16).view(np.uint16), s2h)


def test_serialisation_is_byte_exact():
    data = open(GOLD, "rb").read()
    layers = nq.deserialize_packed_model(data)
    assert nq.serialize_packed_model(layers) == data


def test_write_host_layers_roundtrip(tmp_path):
    layers = nq.read_packed_model(GOLD)
    p = tmp_path / "copy.nqpk"
    nq.write_packed_model(str(p), layers)
    assert p.read_bytes() == open(GOLD, "rb").read()


def test_empty_model():
    data = nq.serialize_packed_model([])
    assert data == b"NQPK" + struct.pack("<II", 1, 0)
    assert nq.deserialize_packed_model(data) == []


@pytest.mark.parametrize("mutate,what", [
    (lambda d: b"NQPX" + d[4:], "magic"),
    (lambda d: d[:4] + struct.pack("<I", 2) + d[8:], "version"),
    (lambda d: d[:-1], "truncated"),
    (lambda d: d + b"\0", "trailing"),
    (lambda d: d[:12] + d[12:16] + d[16:16 + struct.unpack_from("<I", d, 12)[0]]
     + struct.pack("<I", 0) + d[20 + struct.unpack_from("<I", d, 12)[0]:], "zero n"),
])
def test_parse_errors(mutate, what):
    data = open(GOLD, "rb").read()
    with pytest.raises(nq.ParseError):
        nq.deserialize_packed_model(mutate(data))


def test_io_error(tmp_path):
    with pytest.raises(nq.IoError):
        nq.read_packed_model(str(tmp_path / "missing.nqpk"))


def test_matches_reference_serializer_when_available():
    import sys
    sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
    import oracle as O
    if not O.reference_available():
        pytest.skip("reference library not built here")
    ref = O.reference()
    named = [(f"layer{i}", O.synthetic_layer(ref, 0xA000 + i, n, m, r))
             for i, (n, m, r) in enumerate([(33, 65, 31), (17, 200, 64), (128, 8, 5)])]
    ours = nq.serialize_packed_model([(nm, nq.FactorizedLayer(l.n, l.m, l.r, l.u, l.v, l.s1, l.s2))
                                      for nm, l in named])
    assert ours == ref.serialize_nqpk(named)


@pytest.mark.gpu
def test_load_to_device_and_decode():
    import sys
    sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
    import oracle as O
    chk = O.restated()
    dev = nq.load_packed_model(GOLD)
    for (name, d), (_, n, m, r, u, v, s1h, s2h) in zip(dev, golden()):
        back = d.download()
        assert np.array_equal(back.u, u) and np.array_equal(back.v, v)
        lay = O.Layer(n, m, r, u, v, s1h.view(np.float16).astype(np.float64),
                      s2h.view(np.float16).astype(np.float64))
        x = chk.rng(0xC0DE + n).gaussian(m).astype(np.float32)
        want = chk.gemv_packed_f32(lay, x).astype(np.float64)
        got = d.gemv_f32(x).astype(np.float64)
        assert np.linalg.norm(got - want) <= 1e-3 * np.linalg.norm(want), name


@pytest.mark.gpu
def test_write_device_layers_byte_exact(tmp_path):
    dev = nq.load_packed_model(GOLD)
    p = tmp_path / "dev.nqpk"
    nq.write_packed_model(str(p), dev)
    assert p.read_bytes() == open(GOLD, "rb").read()
