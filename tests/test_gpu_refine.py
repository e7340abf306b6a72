"""STE refinement on the device: nqb_ste_refine_layer_host
against the unmodified reference ste_refine (refine.cpp:420-425, run_tuning
:285-384) through oracle/_ref on the pipeline's per-layer group (a one-layer
ToyChain, pipeline.cpp:128-135).  Both run fp64; the device GEMMs sum in a
different order, so the bar is 1e-9 relative on latents and scales, the same
signs, and the same best loss to 1e-9."""
import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu


def toy(seed, n, m, r, b):
    rng = np.random.default_rng(seed)
    lu = rng.standard_normal((n, r))
    lv = rng.standard_normal((m, r))
    s1 = rng.uniform(0.05, 0.2, n)
    s2 = rng.uniform(0.5, 1.5, m)
    x = rng.standard_normal((m, b))
    w = rng.standard_normal((n, m)) * 0.3
    return lu, lv, s1, s2, x, w @ x


def mse(lu, lv, s1, s2, x, t, cw=None):  # refine.cpp:199-212 on the forward of :87-100
    out = s1[:, None] * (np.where(lu < 0, -1.0, 1.0) @ (np.where(lv < 0, -1.0, 1.0).T @ (s2[:, None] * x)))
    d = (t - out) ** 2
    return float((d * (cw[None, :] if cw is not None else 1.0)).sum())


@pytest.mark.parametrize("case", [(24, 16, 6, 20, 4, 4, True, None),
                                  (256, 192, 64, 64, 3, 8, True, None),
                                  (40, 56, 12, 30, 5, 7, False, "weights")])
def test_ste_refine_matches_reference(nq, ref, case):
    n, m, r, b, epochs, batch, cosine, weights = case
    lu, lv, s1, s2, x, t = toy(n * 1000 + m, n, m, r, b)
    cw = np.linspace(0.5, 1.5, b) if weights else None
    cfg = nq.TuneConfig(epochs=epochs, learning_rate=1e-3, batch_size=batch,
                        schedule="cosine" if cosine else "constant", seed=0x5157 + n)
    got, best = nq.ste_refine(nq.FactorizedLatentLayer(lu, lv, s1, s2), x, t, cfg, cw)
    wu, wv, w1, w2, st = ref.ste_refine(lu, lv, s1, s2, x, t, epochs, 1e-3, batch, cosine,
                                        0x5157 + n, cw)
    assert st == 0
    for a, want in ((got.latent_u, wu), (got.latent_v, wv), (got.s1, w1), (got.s2, w2)):
        assert rel(a, want) <= 1e-9
    assert np.array_equal(got.latent_u < 0, wu < 0) and np.array_equal(got.latent_v < 0, wv < 0)
    want_loss = mse(wu, wv, w1, w2, x, t, cw)
    assert abs(best - want_loss) <= 1e-9 * max(want_loss, 1e-300)
    assert best <= mse(lu, lv, s1, s2, x, t, cw) + 1e-12  # never worse than the input
    assert np.any(got.latent_u != lu)  # it did move


def test_ste_refine_errors(nq, ref):
    lu, lv, s1, s2, x, t = toy(5, 8, 6, 3, 10)
    lay = nq.FactorizedLatentLayer(lu, lv, s1, s2)
    with pytest.raises(nq.Error):  # refine.cpp:297-299
        nq.ste_refine(lay, x, t, nq.TuneConfig(epochs=0))
    with pytest.raises(nq.DimensionMismatch):
        nq.ste_refine(lay, x[:5], t, nq.TuneConfig())
    xb = x.copy()
    xb[0, 0] = np.nan
    with pytest.raises(nq.NonFiniteLoss) as ei:  # refine.cpp:306-308
        nq.ste_refine(lay, xb, t, nq.TuneConfig(epochs=1))
    assert np.array_equal(ei.value.best_chain.latent_u, lu)
    _, _, _, _, st = ref.ste_refine(lu, lv, s1, s2, xb, t, 1)
    assert st == nq.NonFiniteLoss.code
