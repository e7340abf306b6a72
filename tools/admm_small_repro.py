import sys, os, time, numpy as np
sys.path.insert(0, os.getcwd())
import bench
import paper_2602_06694_b200 as nq
ca, ws_cpu, r256 = None, None, None
rng = np.random.default_rng(0)
ws = [rng.standard_normal((256, 256)) * 0.02 for _ in range(4)]
r = nq.rank_for_target_bpw(256, 256, 1.0)
try:
    print(bench.admm_small_gpu(nq, ws, r))
except Exception as e:
    import traceback; traceback.print_exc()
