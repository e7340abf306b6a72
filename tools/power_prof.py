import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_06694_b200 as nq
n = int(sys.argv[1]); m = int(sys.argv[2]); k = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = (0.02 * np.random.default_rng(0).standard_normal((n, m))).astype(np.float32).astype(np.float64)
nq.truncated_svd_factors(w, k)
