"""Pins for the oracle's intensity cutoff / pixel percentage and depth profile (reading R14,
P:L299-303; image_set.depth_intensity)."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity import abs_dI  # noqa: F401  (same conftest path setup as the other tests)


def _kth_largest_bruteforce(values, k):
    # order-statistic definition: the value c with #{v >= c} >= k and #{v > c} < k
    vals = [(-math.inf if v != v else float(v)) for v in values]
    for c in sorted(set(vals), reverse=True):
        if sum(v >= c for v in vals) >= k:
            assert sum(v > c for v in vals) < k
            return c
    raise AssertionError


@pytest.mark.parametrize("dtype", ["u16", "f32"])
@pytest.mark.parametrize("fraction", [1e-9, 0.05, 0.25, 0.5, 0.999, 1.0])
def test_select_cutoff_order_statistic(dtype, fraction):
    rng = np.random.default_rng(7)
    img = rng.integers(0, 40, size=(13, 11))  # many ties
    img = img.astype(np.uint16) if dtype == "u16" else (img * 0.37 - 3).astype(np.float32)
    if dtype == "f32":
        img[2, 3] = np.nan
        img[4, 4] = -0.0
    k = min(max(math.ceil(fraction * img.size), 1), img.size)
    c = oracle.select_cutoff(img, fraction)
    assert c == _kth_largest_bruteforce(img.ravel().tolist(), k)
    act = oracle.active_pixels(img, c)
    assert act.sum() >= min(k, int((~np.isnan(img.astype(np.float64))).sum()))  # NaN never passes
    assert (np.nan_to_num(img.astype(np.float64), nan=-np.inf) > c).sum() < k


def test_cutoff_reconstruct_masks_pixels():
    g = synth.geometry("C1")
    stack = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
    full = oracle.reconstruct(g, stack)
    c = oracle.select_cutoff(stack[0], 0.25)
    part = oracle.reconstruct_cutoff(g, stack, c)
    act = stack[0] >= np.float32(c)
    assert 0 < act.sum() < act.size
    assert np.array_equal(part[:, act], full[:, act])
    assert not part[:, ~act].any()
    # the lowest value keeps every pixel
    assert np.array_equal(oracle.reconstruct_cutoff(g, stack, float(stack[0].min())), full)


def _inside_step_stack(g, rng):
    """[S][R][C] stack whose intensity changes only at step pairs whose trapezoid lies inside the
    bin range (exact depths from the independent helper tests/indep.py)."""
    import indep
    S, R, Cc = len(g["wire_xyz"]), g["n_rows"], g["n_cols"]
    lo0 = g["depth_start"] - g["depth_res"] / 2
    hi = g["depth_end"] + g["depth_res"] / 2
    W = g["wire_xyz"]
    d = W[-1] - W[0]
    stack = np.empty((S, R, Cc))
    for j in range(R):
        for i in range(Cc):
            D = np.array([indep.edge_depth_vec(np.repeat(indep.detector_xyz(g, x, j)[None], S, 0), W,
                                               g["wire_axis"], g["wire_radius"], d, g["edge"])
                          for x in (i - 0.5, i + 0.5)])
            lo_c = np.minimum(D[:, :-1].min(0), D[:, 1:].min(0))
            hi_c = np.maximum(D[:, :-1].max(0), D[:, 1:].max(0))
            inside = (lo_c > lo0) & (hi_c < hi)
            steps = np.where(inside, rng.integers(-300, 300, inside.size), 0)
            stack[:, j, i] = 4000.0 + np.concatenate([[0.0], -np.cumsum(steps)])
    return stack


@pytest.mark.parametrize("edge", ["leading", "trailing"])
def test_depth_profile_conservation(edge):
    """image_set.depth_intensity: when every trapezoid lies inside the bins, the profile's
    total is the total intensity change sum_p s (I_0(p) - I_{S-1}(p)) (SURVEY §8(c) conservation,
    summed over the detector); a profile summed over the wrong axis or missing pixels fails it."""
    g = synth.geometry("C1", edge=edge)
    g["n_rows"] = g["n_cols"] = 16  # a 16 x 16 corner of the C1 detector geometry
    g["pitch_col"] = g["pitch_row"] = synth.geometry("C1")["pitch_col"]
    rng = np.random.default_rng(31)
    stack = _inside_step_stack(g, rng)
    prof = oracle.depth_profile(oracle.reconstruct(g, stack))
    assert prof.shape == (oracle.Geometry(g).n_bins,)
    s = 1.0 if edge == "leading" else -1.0
    want = s * (stack[0] - stack[-1]).sum()
    assert abs(want) > 100.0
    assert np.isclose(prof.sum(), want, rtol=1e-12, atol=1e-7)


def test_depth_profile_single_pixel_is_its_depth_column():
    """With one non-constant pixel the profile is that pixel's reconstruction, computed here by the
    independent per-pixel entry point (oracle_reconstruct_pixels)."""
    g = synth.geometry("C1")
    stack = np.full((len(g["wire_xyz"]), g["n_rows"], g["n_cols"]), 1000.0)
    rng = np.random.default_rng(5)
    j, i = 37, 22
    stack[:, j, i] += rng.integers(0, 500, stack.shape[0])
    prof = oracle.depth_profile(oracle.reconstruct(g, stack))
    col = oracle.reconstruct_pixels(g, [j], [i], stack[:, j, i][None])[0]
    assert np.abs(col).max() > 1.0
    assert np.allclose(prof, col, rtol=1e-12, atol=1e-9)
