"""Where a GPU SVD init departs from the reference: truncated_svd_factors of a
fixture's W on the device (run on the GPU box) or through oracle/_ref (here),
saved to an .npz; `compare` prints the first deflation steps whose factor
columns differ.  python tools/svd_diag.py gpu|ref|compare NAME"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

mode, name = sys.argv[1], sys.argv[2]
g = np.load(os.path.join(ROOT, "tests", "golden", f"admm_{name}.npz"))
n, m, r = int(g["n"]), int(g["m"]), int(g["r"])
if mode in ("gpu", "ref"):
    w = O.synthetic_weight(O.restated(), int(g["seed"]), n, m)
    if mode == "gpu":
        import paper_2602_06694_b200 as nq
        u, v = nq.truncated_svd_factors(w, r)
    else:
        u, v = O.reference().truncated_svd_factors(w, r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", f"svd_{mode}_{name}.npz"), u=u, v=v)
else:
    a = np.load(os.path.join(ROOT, "gpurun_out", f"svd_gpu_{name}.npz"))
    b = np.load(os.path.join(ROOT, "gpurun_out", f"svd_ref_{name}.npz"))
    du = np.abs(a["u"] - b["u"]).max(0) / (np.abs(b["u"]).max(0) + 1e-300)
    dv = np.abs(a["v"] - b["v"]).max(0) / (np.abs(b["v"]).max(0) + 1e-300)
    d = np.maximum(du, dv)
    print("max rel diff per step: first 10", d[:10])
    for thr in (1e-12, 1e-9, 1e-6, 1e-3):
        idx = np.nonzero(d > thr)[0]
        print(f"first step above {thr:g}: {idx[0] if idx.size else None} ({idx.size} steps)")
