"""Pins for the oracle's trapezoid CDF and per-pair deposit.

* H(z) against numerical integration of the unit-height trapezoid (scipy.quad);
* per-bin weights against numerically integrated bin overlaps, including the
  out-of-range drop (reading R7) and the degenerate delta (reading R8);
* POINT mode (box) against the textbook interval-overlap fraction;
* one whole step pair against brute-force fine subdivision of the pixel width x
  the wire interval with exact (independently computed) tangent depths.
"""
import math

import numpy as np
import pytest
from scipy.integrate import quad

import indep
import oracle
import synth


def _rand_corners(rng):
    kind = rng.integers(0, 5)
    z = np.sort(rng.uniform(-5, 5, 4))
    if kind == 1:
        z[1] = z[0]  # no rising ramp
    elif kind == 2:
        z[3] = z[2]  # no falling ramp
    elif kind == 3:
        z[2] = z[1]  # triangle
    elif kind == 4:
        z[1] = z[0]
        z[3] = z[2]  # box
    return z


def test_cdf_matches_numeric_integration():
    rng = np.random.default_rng(10)
    for _ in range(300):
        z = _rand_corners(rng)
        A = 0.5 * (z[3] + z[2] - z[1] - z[0])
        for x in list(rng.uniform(-6, 6, 5)) + list(z):
            pts = [p for p in z if -10 < p < x]
            want = quad(lambda t: float(indep.trapezoid_pdf(t, z)), -10, x, points=pts or None, limit=200)[0] \
                if x > -10 else 0.0
            assert abs(oracle.trapezoid_cdf(z, x) - want) < 1e-9, (z, x)
        assert abs(oracle.trapezoid_cdf(z, 99.0) - A) < 1e-12


def test_deposit_weights_match_integrated_overlap():
    rng = np.random.default_rng(11)
    start, dz, M = -3.0, 0.7, 9  # bins [-3.35, 2.95)
    lo0, hiM = start - dz / 2, start + (M - 0.5) * dz
    for _ in range(200):
        z = _rand_corners(rng)
        perm = rng.permutation(4)  # the oracle must sort the corners itself
        dI = rng.uniform(-100, 100)
        got = oracle.deposit_pair(dI, z[perm], start, dz, M)
        A = 0.5 * (z[3] + z[2] - z[1] - z[0])
        want = np.zeros(M)
        for m in range(M):
            lo, hi = start + (m - 0.5) * dz, start + (m + 0.5) * dz
            pts = [p for p in z if lo < p < hi]
            want[m] = dI * quad(lambda t: float(indep.trapezoid_pdf(t, z)), lo, hi, points=pts or None,
                                limit=200)[0] / A
        assert np.allclose(got, want, atol=1e-8 * abs(dI), rtol=0), (z, got, want)
        # mass: all of dI when the trapezoid is inside the bin range, else only the inside part
        inside = lo0 <= z[0] and z[3] <= hiM
        if inside:
            assert abs(got.sum() - dI) < 1e-10 * abs(dI)


def test_point_mode_box_is_interval_overlap():
    rng = np.random.default_rng(12)
    start, dz, M = 0.0, 1.0, 12
    for _ in range(200):
        a, b = np.sort(rng.uniform(-1, 12, 2))
        got = oracle.deposit_pair(1.0, [b, a, a, b], start, dz, M)
        lo = start + (np.arange(M) - 0.5) * dz
        want = np.clip(np.minimum(lo + dz, b) - np.maximum(lo, a), 0, None) / (b - a)
        assert np.allclose(got, want, atol=1e-12)


def test_degenerate_delta_goes_to_containing_bin():
    start, dz, M = 0.0, 1.0, 5  # bins [-0.5,0.5) [0.5,1.5) ...
    for z, m in [(0.2, 0), (0.5, 1), (-0.5, 0), (4.49, 4)]:
        got = oracle.deposit_pair(3.0, [z] * 4, start, dz, M)
        want = np.zeros(M)
        want[m] = 3.0
        assert np.array_equal(got, want), (z, got)
    assert not oracle.deposit_pair(3.0, [4.5] * 4, start, dz, M).any()  # outside: dropped
    assert not oracle.deposit_pair(3.0, [-0.51] * 4, start, dz, M).any()


def test_out_of_range_parts_are_dropped():
    # box [-1, 1] over bins starting at lo_0 = -0.5: only [-0.5, 1] is inside
    got = oracle.deposit_pair(2.0, [-1, -1, 1, 1], 0.0, 1.0, 3)
    assert np.allclose(got, [1.0, 0.5, 0.0])


@pytest.mark.parametrize("pixel_model", ["finite", "point"])
def test_pair_against_brute_force_subdivision(pixel_model):
    """Fine subdivision of pixel width (u) x wire interval (t), exact tangent depths
    from tests/indep.py, histogrammed into the bins -> converges to the trapezoid
    weights (SURVEY.md §8(c) Pins; the trapezoid is first-order exact)."""
    g = synth.geometry("C2", pixel_model=pixel_model)
    g["depth_res"] = 0.25
    g["depth_start"], g["depth_end"] = -50.0, 50.0
    M = oracle.Geometry(g).n_bins
    W = g["wire_xyz"]
    d = W[-1] - W[0]
    rng = np.random.default_rng(13)
    n_u, n_t = 1200, 1200
    for (j, i) in [(0, 0), (100, 255), (511, 511), (300, 40)]:
        # pick a pair whose depth interval lands inside the bins
        Qc = indep.detector_xyz(g, i, j)
        Dk = indep.edge_depth_vec(np.repeat(Qc[None], len(W), 0), W, g["wire_axis"], g["wire_radius"], d)
        k = int(np.argmin(np.abs(Dk - rng.uniform(-30, 30))))
        series = np.zeros(len(W))
        series[: k + 1] = 1.0  # dI = 1 only at pair k
        got = oracle.reconstruct_pixels(g, [j], [i], series[None])[0]
        # brute force
        if pixel_model == "finite":
            us = i - 0.5 + (np.arange(n_u) + 0.5) / n_u
        else:
            us = np.array([float(i)])
            n_t = 40000  # 1-D: a fine t grid alone
        ts = (np.arange(n_t) + 0.5) / n_t
        Qs = np.array([indep.detector_xyz(g, u, j) for u in us])
        Wt = W[k][None] + ts[:, None] * (W[k + 1] - W[k])[None]
        QQ = np.repeat(Qs, len(ts), 0)
        WW = np.tile(Wt, (len(us), 1))
        D = indep.edge_depth_vec(QQ, WW, g["wire_axis"], g["wire_radius"], d)
        lo0 = g["depth_start"] - g["depth_res"] / 2
        idx = np.floor((D - lo0) / g["depth_res"]).astype(int)
        want = np.bincount(idx[(idx >= 0) & (idx < M)], minlength=M)[:M] / len(D)
        assert abs(got.sum() - 1.0) < 1e-9
        # measured 1.5e-5..6e-5; a half-pixel centre shift gives 3e-2..8e-2
        assert np.abs(got - want).max() < 3e-4, (j, i, k, np.abs(got - want).max())
        # the binned first moment (mean depth) agrees to a small fraction of a bin
        centres = g["depth_start"] + np.arange(M) * g["depth_res"]
        assert abs(got @ centres - want @ centres) < 0.01 * g["depth_res"]
