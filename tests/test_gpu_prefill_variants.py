"""The prefill kernel variants, each through the same parity tests.

Kernel selection is read from the environment once per process, so each variant
runs the prefill parity tests of test_gpu_forward.py in a subprocess:
* CTA pair (`cta_group::2`) with 128 and with 256 rows per CTA, with and without split-K;
* the single-CTA SS kernel;
* the A-in-TMEM (TS) kernel."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"NQB_PREFILL_ROWS": "128"}, {"NQB_PREFILL_ROWS": "256"},
                                 {"NQB_PREFILL_SPLITK": "3"}, {"NQB_PREFILL_N": "208"},
                                 {"NQB_PREFILL_ROWS": "128", "NQB_PREFILL_N": "208"},
                                 {"NQB_PREFILL_ROWS": "128", "NQB_PREFILL_SPLITK": "2"},
                                 {"NQB_PREFILL_2SM": "0"}, {"NQB_PREFILL_2SM": "0", "NQB_PREFILL_TS": "1"}],
                         ids=["pair128", "pair256", "pair_splitk3", "pair_n208", "pair128_n208", "pair128_splitk2",
                              "ss", "ts"])
def test_prefill_variant_parity(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_forward.py"), "-k", "prefill or gemm"],
                       env={**os.environ, **env}, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
