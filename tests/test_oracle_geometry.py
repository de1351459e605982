"""Pins for the oracle's geometry ("Pins").

Each check compares the oracle with something other than itself: scipy's
rotation-vector routine, the tangent-line quadratic (tests/indep.py), the
pixel-above-the-wire closed form, the r -> 0 similar-triangles limit and the
invariances of the tangent construction.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
import indep

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_rodrigues_matches_scipy():
    rng = np.random.default_rng(1)
    for _ in range(20):
        R = rng.normal(size=3) * rng.uniform(0.1, 3.0)
        assert np.allclose(oracle.rodrigues(R), indep.det_rotation(R), atol=1e-14)
    assert np.allclose(oracle.rodrigues([0, 0, 0]), np.eye(3))
    # SURVEY appendix frame check: -(2pi/3)/sqrt3 (1,1,1) maps x'->z, y'->x, z'->y
    rho = oracle.rodrigues(-(2 * math.pi / 3) / math.sqrt(3) * np.ones(3))
    assert np.allclose(rho @ [1, 0, 0], [0, 0, 1], atol=1e-14)
    assert np.allclose(rho @ [0, 1, 0], [1, 0, 0], atol=1e-14)
    assert np.allclose(rho @ [0, 0, 1], [0, 1, 0], atol=1e-14)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_detector_point_convention(cfg):
    g = synth.geometry(cfg)
    for (x, j) in [(0, 0), (g["n_cols"] - 1, 3), (-0.5, 7), (g["n_cols"] / 3 + 0.5, g["n_rows"] - 1)]:
        assert np.allclose(oracle.detector_point(g, x, j), indep.detector_xyz(g, x, j), rtol=0, atol=1e-8)
    # adjacent columns are exactly one pitch apart
    a, b = oracle.detector_point(g, 10, 5), oracle.detector_point(g, 11, 5)
    assert abs(np.linalg.norm(b - a) - g["pitch_col"]) < 1e-7


def _random_setup(rng):
    Q = np.array([rng.uniform(-2e5, 2e5), rng.uniform(4e5, 6e5), rng.uniform(-2e5, 2e5)])
    W = np.array([rng.uniform(-50, 50), rng.uniform(100, 600), rng.uniform(-300, 300)])
    axis = np.array([1.0, rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1)])
    axis /= np.linalg.norm(axis)
    beam = np.array([rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05), 1.0])
    beam /= np.linalg.norm(beam)
    origin = rng.uniform(-20, 20, size=3)
    r = rng.uniform(5, 60)
    return Q, W, axis, r, beam, origin


def test_tangent_depth_equals_quadratic_roots():
    rng = np.random.default_rng(2)
    for _ in range(200):
        Q, W, axis, r, beam, origin = _random_setup(rng)
        roots, _, _ = indep.tangent_roots(Q, W, axis, r, beam, origin)
        got = sorted(oracle.tangent_depth(Q, W, axis, r, s, beam, origin) for s in (+1.0, -1.0))
        assert np.allclose(got, roots, rtol=1e-11, atol=1e-9), (got, roots)


def test_leading_edge_is_the_side_facing_the_motion():
    """sigma from oracle_edge_sigma picks the contact point on the wire side facing d (leading)."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        Q, W0, axis, r, beam, origin = _random_setup(rng)
        d = np.array([0.0, 1.0, 1.0]) / math.sqrt(2) + rng.normal(size=3) * 0.05
        Wl = W0 + 700 * d
        for edge in ("leading", "trailing"):
            sig = oracle.edge_sigma(Q, W0, Wl, axis, edge)
            for W in (W0, W0 + 350 * d):
                want = indep.edge_depth(Q, W, axis, r, Wl - W0, edge, beam, origin)
                got = oracle.tangent_depth(Q, W, axis, r, sig, beam, origin)
                assert abs(got - want) < 1e-8 * max(1.0, abs(want))


def test_pixel_above_wire_closed_form():
    """Pixel directly above the wire centre, beam along z: D = z_w +- Y r / sqrt((Y-y_w)^2 - r^2).
    Golden numbers: tests/golden/pixel_above_wire.json (SURVEY.md §8(c) Pins (ii))."""
    with open(os.path.join(GOLD, "pixel_above_wire.json")) as f:
        gold = json.load(f)
    Y, yw, r = gold["Y"], gold["y_w"], gold["r"]
    for zw in (0.0, 17.5, -230.0):
        Q = np.array([0.0, Y, zw])
        W = np.array([0.0, yw, zw])
        closed = Y * r / math.sqrt((Y - yw) ** 2 - r * r)
        got = sorted(oracle.tangent_depth(Q, W, [1, 0, 0], r, s, [0, 0, 1], [0, 0, 0]) for s in (1, -1))
        assert np.allclose(got, [zw - closed, zw + closed], rtol=0, atol=1e-9)
        if zw == 0.0:
            assert abs(got[1] - gold["D_plus"]) < 5e-6 and abs(got[0] - gold["D_minus"]) < 5e-6
        # leading edge for motion along +H = (0,1,1)/sqrt2 is the downstream (larger-z) edge
        sig = oracle.edge_sigma(Q, W, W + np.array([0, 1, 1.0]), np.array([1.0, 0, 0]), "leading")
        assert abs(oracle.tangent_depth(Q, W, [1, 0, 0], r, sig, [0, 0, 1], [0, 0, 0]) - (zw + closed)) < 1e-9


def test_r_to_zero_similar_triangles():
    rng = np.random.default_rng(4)
    for _ in range(50):
        Q, W, axis, _, beam, origin = _random_setup(rng)
        # r -> 0: the line through Q and the wire centre W meets the beam (2-D, perpendicular to axis)
        a, u, v = indep._frame(axis)
        P = lambda z: origin + z * beam
        q2 = np.array([(Q - W) @ u, (Q - W) @ v])
        f = lambda z: q2[0] * ((P(z) - W) @ v) - q2[1] * ((P(z) - W) @ u)
        z0 = -f(0.0) / (f(1.0) - f(0.0))  # f is affine in z
        for r in (1e-3, 1e-4):
            for s in (1, -1):
                D = oracle.tangent_depth(Q, W, axis, r, s, beam, origin)
                assert abs(D - z0) < 5e3 * r  # |dD/dr| ~ L_beam/L_wire-ish, bounded


def test_tangent_invariances():
    rng = np.random.default_rng(5)
    for _ in range(50):
        Q, W, axis, r, beam, origin = _random_setup(rng)
        D = oracle.tangent_depth(Q, W, axis, r, 1.0, beam, origin)
        # rigid motion of everything
        Rm = indep.det_rotation(rng.normal(size=3))
        t = rng.normal(size=3) * 100
        D2 = oracle.tangent_depth(Rm @ Q + t, Rm @ W + t, Rm @ axis, r, 1.0, Rm @ beam, Rm @ origin + t)
        assert abs(D2 - D) < 1e-7 * max(1, abs(D))
        # translations along the wire axis
        assert abs(oracle.tangent_depth(Q + 77.0 * axis, W, axis, r, 1.0, beam, origin) - D) < 1e-7 * max(1, abs(D))
        assert abs(oracle.tangent_depth(Q, W - 31.0 * axis, axis, r, 1.0, beam, origin) - D) < 1e-7 * max(1, abs(D))
        # sigma <-> -sigma equals r <-> -r
        assert abs(oracle.tangent_depth(Q, W, axis, -r, -1.0, beam, origin) - D) < 1e-9 * max(1, abs(D))
        # moving the depth origin along the beam shifts depth by the same amount
        assert abs(oracle.tangent_depth(Q, W, axis, r, 1.0, beam, origin + 5.0 * beam) - (D - 5.0)) < 1e-7 * max(1, abs(D))


def test_degenerate_geometry_is_nan():
    # pixel inside the wire cylinder -> no tangent
    assert math.isnan(oracle.tangent_depth([0, 10, 0], [0, 0, 0], [1, 0, 0], 26, 1, [0, 0, 1], [0, 0, 0]))
    # tangent plane parallel to the beam: pixel and wire on the beam line side, n.k = 0
    # (pixel in the plane y = r, which is tangent to the wire and contains the beam direction)
    d = oracle.tangent_depth([0, 26, 1000], [0, 0, 0], [1, 0, 0], 26, -1, [0, 0, 1], [0, 0, 0])
    assert math.isnan(d)
    assert not math.isnan(oracle.tangent_depth([0, 26, 1000], [0, 0, 0], [1, 0, 0], 26, 1, [0, 0, 1], [0, 0, 0]))
