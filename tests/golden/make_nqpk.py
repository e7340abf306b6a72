"""Writes tests/golden/nqpk_small.nqpk with the UNMODIFIED reference serializer
(serialize_packed_model, io.cpp:139-158, via oracle/_ref) and the layers it holds
to tests/golden/nqpk_small.npz, so the NQPK tests can check parsing and
byte-exact serialisation without the reference at run time.

Run here (where /root/reference exists):  python tests/golden/make_nqpk.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

# (name, n, m, r, seed): ragged ranks (tails of the last word), a multi-byte UTF-8 name
LAYERS = [("blocks.0.attn.q", 40, 70, 37, 0x9B01), ("blocks.0.mlp.gate", 64, 48, 11, 0x9B02),
          ("résidu/down", 96, 128, 70, 0x9B03)]


def main():
    ref = O.reference()
    named = [(nm, O.synthetic_layer(ref, seed, n, m, r)) for nm, n, m, r, seed in LAYERS]
    data = ref.serialize_nqpk(named)
    with open(os.path.join(HERE, "nqpk_small.nqpk"), "wb") as f:
        f.write(data)
    arrays = {}
    for i, (nm, l) in enumerate(named):
        arrays[f"u{i}"], arrays[f"v{i}"] = l.u, l.v
        arrays[f"s1h{i}"] = ref.double_to_half(l.s1)
        arrays[f"s2h{i}"] = ref.double_to_half(l.s2)
        arrays[f"dims{i}"] = np.array([l.n, l.m, l.r], np.uint32)
    arrays["names"] = np.array([nm for nm, *_ in LAYERS])
    np.savez_compressed(os.path.join(HERE, "nqpk_small.npz"), **arrays)
    print(f"nqpk_small.nqpk: {len(data)} bytes, {len(named)} layers")


if __name__ == "__main__":
    main()
