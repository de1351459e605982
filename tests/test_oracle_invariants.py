"""Whole-oracle pins (SURVEY.md §8(c) "Whole oracle"; BASELINE.json north_star):

(a) conservation: per pixel, sum over bins = s (I_0 - I_{S-1}) when every
    trapezoid lies inside the bin range;
(b) a constant background added to every step changes nothing;
(c) linearity in the stack;
(d) step reversal <-> trailing identity: the leading reconstruction of the
    step-reversed scan equals the (sign-normalised) trailing reconstruction;
(e) forward-model round trip with an independent occlusion model;
plus the NaN-corner skip rule and the raw/normalised trailing sign.
"""
import numpy as np
import pytest

import indep
import oracle
import synth


def _edge_depths(g, j, i):
    """Exact depths of the back/front pixel edges at every wire step (independent helper)."""
    W = g["wire_xyz"]
    d = W[-1] - W[0]
    out = []
    for x in (i - 0.5, i + 0.5):
        Q = indep.detector_xyz(g, x, j)
        out.append(indep.edge_depth_vec(np.repeat(Q[None], len(W), 0), W, g["wire_axis"], g["wire_radius"], d,
                                        g["edge"]))
    return np.array(out)  # [2, S]


@pytest.mark.parametrize("edge", ["leading", "trailing"])
def test_conservation_when_inside_bin_range(edge):
    g = synth.geometry("C2", edge=edge)
    rng = np.random.default_rng(20)
    lo0 = g["depth_start"] - g["depth_res"] / 2
    hi = g["depth_end"] + g["depth_res"] / 2
    pix = [(0, 0), (7, 511), (256, 256), (500, 3), (123, 321)]
    series = []
    for (j, i) in pix:
        D = _edge_depths(g, j, i)
        lo_c = np.minimum(D[:, :-1].min(0), D[:, 1:].min(0))
        hi_c = np.maximum(D[:, :-1].max(0), D[:, 1:].max(0))
        inside = (lo_c > lo0) & (hi_c < hi)
        assert inside.sum() > 10
        steps = np.where(inside, rng.integers(-500, 500, inside.size), 0)
        I = 5000.0 + np.concatenate([[0.0], -np.cumsum(steps)])
        series.append(I)
    series = np.array(series)
    out = oracle.reconstruct_pixels(g, [p[0] for p in pix], [p[1] for p in pix], series)
    s = 1.0 if edge == "leading" else -1.0
    want = s * (series[:, 0] - series[:, -1])
    assert np.allclose(out.sum(1), want, rtol=1e-12, atol=1e-9)


def test_constant_background_and_linearity():
    g = synth.geometry("C1")
    maps = synth.make_maps("C1")
    X = synth.stack_numpy(maps, "f64", noise=True)
    rng = np.random.default_rng(21)
    Y = rng.integers(0, 3000, X.shape).astype(np.float64)
    oX, oY = oracle.reconstruct(g, X), oracle.reconstruct(g, Y)
    assert np.abs(oX).max() > 1.0
    assert np.array_equal(oracle.reconstruct(g, X + 777.0), oX)  # integer data: exact
    a, b = 3.0, -2.0
    assert np.allclose(oracle.reconstruct(g, a * X + b * Y), a * oX + b * oY, rtol=0, atol=1e-9 * np.abs(oY).max())


@pytest.mark.parametrize("pixel_model", ["finite", "point"])
def test_step_reversal_equals_trailing(pixel_model):
    g = synth.geometry("C1", pixel_model=pixel_model)
    maps = synth.make_maps("C1")
    X = synth.stack_numpy(maps, "f64", noise=True)
    trail = oracle.reconstruct(dict(g, edge="trailing"), X)
    g_rev = dict(g, wire_xyz=g["wire_xyz"][::-1].copy())
    lead_rev = oracle.reconstruct(g_rev, X[::-1].copy())
    assert np.abs(trail).max() > 1.0
    assert np.allclose(lead_rev, trail, rtol=0, atol=1e-9)
    raw = oracle.reconstruct(dict(g, edge="trailing"), X, raw_sign=True)
    assert np.array_equal(raw, -trail)


def test_nan_corner_pairs_are_skipped():
    """A wire position that swallows the pixel (L <= r) makes those pairs NaN -> skipped,
    exactly as if their dI were zero."""
    g = synth.geometry("C1")
    j, i = 5, 9
    Q = indep.detector_xyz(g, i, j)
    W = g["wire_xyz"].copy()
    W[7] = Q + np.array([0.0, 1.0, 0.0])  # inside the wire cylinder around the pixel
    g2 = dict(g, wire_xyz=W)
    rng = np.random.default_rng(22)
    I = rng.integers(0, 1000, g["wire_xyz"].shape[0]).astype(float)
    got = oracle.reconstruct_pixels(g2, [j], [i], I[None])
    I2 = I.copy()
    # pairs 6 and 7 touch step 7: zero their dI by flattening, keeping the rest
    dI = I[:-1] - I[1:]
    dI[6] = dI[7] = 0.0
    I2 = np.concatenate([[I[0]], I[0] - np.cumsum(dI)])
    want = oracle.reconstruct_pixels(g2, [j], [i], I2[None])
    assert np.allclose(got, want, atol=1e-9)
    assert np.isfinite(got).all()


@pytest.mark.parametrize("edge", ["leading", "trailing"])
def test_forward_model_round_trip(edge):
    """Independent occlusion model (tests/indep.occluded: segment source->pixel within r of
    the wire axis) generates the intensities of a thin slab source; the reconstruction
    must put the slab's mass in the slab's bins."""
    g = synth.geometry("C2", edge=edge)
    g["wire_xyz"] = synth.wire_positions(801)
    g["depth_res"] = 0.5
    z_a, z_b = -10.3, -6.9
    n_z, n_u = 240, 6
    zs = z_a + (np.arange(n_z) + 0.5) / n_z * (z_b - z_a)
    W = g["wire_xyz"]
    pix = [(0, 0), (256, 256), (511, 511), (100, 400)]
    series = []
    for (j, i) in pix:
        us = i - 0.5 + (np.arange(n_u) + 0.5) / n_u
        Qs = np.array([indep.detector_xyz(g, u, j) for u in us])
        P = np.zeros((n_z, 3))
        P[:, 2] = zs
        PP = np.repeat(P, n_u, 0)
        QQ = np.tile(Qs, (n_z, 1))
        I = np.empty(len(W))
        for k in range(len(W)):
            blocked = indep.occluded(PP, QQ, W[k][None], g["wire_axis"], g["wire_radius"])
            I[k] = (~blocked).sum() / n_u
        series.append(I)
    series = np.array(series)
    out = oracle.reconstruct_pixels(g, [p[0] for p in pix], [p[1] for p in pix], series)
    centres = g["depth_start"] + np.arange(out.shape[1]) * g["depth_res"]
    in_slab = (centres > z_a - g["depth_res"]) & (centres < z_b + g["depth_res"])
    for p in range(len(pix)):
        frac = out[p, in_slab].sum() / n_z
        assert frac > 0.95, (pix[p], frac)  # measured 0.972..0.998
        assert in_slab[np.argmax(out[p])]
