"""Pins of the oracle's per-step intensity normalisation (SURVEY.md §8(f)4 "per-step I0
normalisation"; reading R17: dI_k = s (w_k I_k - w_{k+1} I_{k+1}), w_k the step's
normalisation weight, e.g. I0_ref / I0_k from the beam monitor).

Each pin would fail for a weight applied to the difference instead of the intensities
(w_k (I_k - I_{k+1})), a weight shifted by one step, or a weight dropped on one side."""
import numpy as np
import pytest

import oracle
import synth
from test_oracle_invariants import _edge_depths


def test_constant_weight_scales_the_reconstruction():
    g = synth.geometry("C1")
    X = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
    S = X.shape[0]
    plain = oracle.reconstruct(g, X)
    scaled = oracle.reconstruct(dict(g, step_weight=np.full(S, 2.5)), X)
    assert np.abs(plain).max() > 1.0
    assert np.allclose(scaled, 2.5 * plain, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("edge", ["leading", "trailing", "both"])
def test_weights_normalise_the_images_before_differencing(edge):
    """Weighted reconstruction of I = the unweighted reconstruction of the normalised images w_k I_k."""
    g = synth.geometry("C1", edge=edge)
    X = synth.stack_numpy(synth.make_maps("C1"), "u16", noise=True)
    S = X.shape[0]
    w = np.random.default_rng(5).uniform(0.8, 1.25, S)
    got = oracle.reconstruct(dict(g, step_weight=w), X)
    want = oracle.reconstruct(g, X.astype(np.float64) * w[:, None, None])
    assert np.abs(got - oracle.reconstruct(g, X)).max() > 1.0  # the weights matter
    assert np.allclose(got, want, rtol=1e-12, atol=1e-8)


def test_weighted_conservation():
    """Sum over bins = s (w_0 I_0 - w_{S-1} I_{S-1}) when every pair with a nonzero weighted
    difference lies inside the bin range (weights != 1 only where the pixel's trapezoids are inside)."""
    g = synth.geometry("C2")
    lo0 = g["depth_start"] - g["depth_res"] / 2
    hi = g["depth_end"] + g["depth_res"] / 2
    rng = np.random.default_rng(11)
    for (j, i) in [(7, 511), (256, 256), (123, 321)]:
        D = _edge_depths(g, j, i)
        lo_c = np.minimum(D[:, :-1].min(0), D[:, 1:].min(0))
        hi_c = np.maximum(D[:, :-1].max(0), D[:, 1:].max(0))
        inside = (lo_c > lo0) & (hi_c < hi)  # pair k
        S = D.shape[1]
        k_in = np.where(inside)[0]
        a, b = k_in[0] + 1, k_in[-1]  # steps whose both pairs are inside
        assert b - a > 10 and inside[a - 1:b + 1].all()
        w = np.ones(S)
        w[a:b + 1] = rng.uniform(0.7, 1.3, b + 1 - a)
        steps = np.where(inside, rng.integers(-500, 500, inside.size), 0)
        I = 5000.0 + np.concatenate([[0.0], -np.cumsum(steps)])
        out = oracle.reconstruct_pixels(dict(g, step_weight=w), [j], [i], I[None])
        assert np.isclose(out.sum(), w[0] * I[0] - w[-1] * I[-1], rtol=1e-12, atol=1e-8)
