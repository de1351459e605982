"""Pins of the oracle's both-edges mode (reading R16): the leading edge takes each
step's intensity decrease max(I_k - I_{k+1}, 0) with the leading-edge geometry, the trailing
edge takes the increase max(I_{k+1} - I_k, 0) (the sign-normalised trailing dI, reading R2) with
the trailing-edge geometry, and the two reconstructions add.

The pins go through the single-edge oracle (pinned in test_oracle_*.py) on derived stacks, or
through the independent occlusion model (tests/indep.py), never through the both-mode code."""
import numpy as np
import pytest

import indep
import oracle
import synth


def _split(stack):
    """D keeps only the decreases of `stack` along the step axis, U only the increases."""
    d = np.diff(stack.astype(np.float64), axis=0)
    z = np.zeros_like(stack[:1], dtype=np.float64)
    D = stack[:1] + np.concatenate([z, np.cumsum(np.minimum(d, 0.0), axis=0)])
    U = stack[:1] + np.concatenate([z, np.cumsum(np.maximum(d, 0.0), axis=0)])
    return D, U


@pytest.mark.parametrize("pixel_model", ["finite", "point"])
def test_both_is_leading_of_decreases_plus_trailing_of_increases(pixel_model):
    """both(I) = lead(D) + trail(U): D, U the decreasing / increasing parts of I.  Fails for a
    wrong trailing sign, a missing or reversed clamp, or swapped edge geometries."""
    gb = synth.geometry("C1", edge="both", pixel_model=pixel_model)
    gl = synth.geometry("C1", edge="leading", pixel_model=pixel_model)
    gt = synth.geometry("C1", edge="trailing", pixel_model=pixel_model)
    rng = np.random.default_rng(16)
    stack = 5000.0 + rng.integers(-400, 400, (21, 64, 64)).astype(np.float64)
    D, U = _split(stack)
    both = oracle.reconstruct(gb, stack)
    ref = oracle.reconstruct(gl, D) + oracle.reconstruct(gt, U)
    assert np.abs(ref).max() > 100
    assert np.allclose(both, ref, rtol=1e-12, atol=1e-9)
    # and it is neither single edge, nor their plain sum
    assert not np.allclose(both, oracle.reconstruct(gl, stack), atol=1.0)
    assert not np.allclose(both, oracle.reconstruct(gl, stack) + oracle.reconstruct(gt, stack), atol=1.0)


def test_monotone_stacks_reduce_to_one_edge():
    """A stack that only decreases is the leading reconstruction, one that only increases the
    trailing one -- bit for bit (the other edge's terms are all skipped)."""
    rng = np.random.default_rng(17)
    steps = rng.integers(0, 300, (20, 64, 64)).astype(np.float64)
    down = 9000.0 - np.concatenate([np.zeros((1, 64, 64)), np.cumsum(steps, axis=0)])
    up = 1000.0 + np.concatenate([np.zeros((1, 64, 64)), np.cumsum(steps, axis=0)])
    gb = synth.geometry("C1", edge="both")
    assert np.array_equal(oracle.reconstruct(gb, down), oracle.reconstruct(synth.geometry("C1"), down))
    assert np.array_equal(oracle.reconstruct(gb, up), oracle.reconstruct(synth.geometry("C1", edge="trailing"), up))


def test_forward_model_slab_counts_twice():
    """A thin slab source seen through the independent occlusion model (tests/indep.occluded):
    its intensity drops while the wire's leading edge covers the rays and comes back when the
    trailing edge uncovers them, so the both-edges reconstruction puts twice the slab's mass in
    the slab's bins (each single edge: once; a single edge also deposits the other edge's change,
    with the opposite sign, at a ghost depth)."""
    g = synth.geometry("C2", edge="both")
    g["wire_xyz"] = synth.wire_positions(801, t_range=(-100.0, 1500.0))
    g["depth_res"] = 0.5
    z_a, z_b = -10.3, -6.9
    n_z, n_u = 160, 4
    zs = z_a + (np.arange(n_z) + 0.5) / n_z * (z_b - z_a)
    W = g["wire_xyz"]
    pix = [(256, 256), (100, 400)]
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
            I[k] = (~indep.occluded(PP, QQ, W[k][None], g["wire_axis"], g["wire_radius"])).sum() / n_u
        series.append(I)
    series = np.array(series)
    # the scan starts and ends with every ray open: one full cover-uncover cycle
    assert np.allclose(series[:, 0], n_z) and np.allclose(series[:, -1], n_z) and series.min() < 1
    rows, cols = [p[0] for p in pix], [p[1] for p in pix]
    out = oracle.reconstruct_pixels(g, rows, cols, series)
    centres = g["depth_start"] + np.arange(out.shape[1]) * g["depth_res"]
    in_slab = (centres > z_a - g["depth_res"]) & (centres < z_b + g["depth_res"])
    for p in range(len(pix)):
        assert 1.9 < out[p, in_slab].sum() / n_z <= 2.0 + 1e-9, (pix[p], out[p, in_slab].sum() / n_z)
        assert in_slab[np.argmax(out[p])]
    for edge in ("leading", "trailing"):
        g1 = dict(g, edge=edge)
        one = oracle.reconstruct_pixels(g1, rows, cols, series)
        for p in range(len(pix)):
            assert 0.9 < one[p, in_slab].sum() / n_z <= 1.0 + 1e-9  # measured 0.945 .. 0.99
