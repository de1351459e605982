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


def test_depth_profile_conserves_intensity():
    g = synth.geometry("C1")
    stack = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=False)
    out = oracle.reconstruct(g, stack)
    prof = oracle.depth_profile(out)
    assert prof.shape == (out.shape[0],)
    # all depth-resolved intensity is deposited: profile total = sum of the deposited pixel totals
    assert np.isclose(prof.sum(), out.sum(), rtol=1e-12)
    assert np.allclose(prof, [out[m].sum() for m in range(out.shape[0])], rtol=1e-12)
