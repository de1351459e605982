"""The shared input generator: determinism, numpy == torch bit for bit, row bands,
and that the synthetic wire travel sweeps the whole bin range at every pixel."""
import numpy as np
import pytest
import torch

import oracle
import synth


@pytest.mark.parametrize("dtype", ["u16", "f32"])
def test_numpy_torch_identical(dtype):
    maps = synth.make_maps("C1")
    for noise in (False, True):
        a = synth.stack_numpy(maps, dtype, noise=noise)
        b = synth.stack_torch(maps, dtype, "cpu", noise=noise).numpy()
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_pixel_series_and_row_band_match_full_stack():
    maps = synth.make_maps("C2")
    full = synth.stack_numpy(maps, "u16", noise=True)
    band = synth.stack_numpy(maps, "u16", noise=True, rows=(100, 140))
    assert np.array_equal(full[:, 100:140], band)
    js, is_ = np.array([0, 5, 511, 200]), np.array([0, 511, 3, 250])
    ser = synth.pixel_series(maps, js, is_, "u16", noise=True)
    assert np.array_equal(ser, full[:, js, is_].T)


def test_maps_deterministic_and_peaked():
    a, b = synth.make_maps("C3"), synth.make_maps("C3")
    for f in ("bg", "amp", "ka", "w", "kt"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert (a.amp > 0).sum() > 100 and (a.w >= 1).all()
    c5 = synth.make_maps("C5")
    frac = (c5.amp > 0).mean()
    assert 0.005 < frac < 0.03  # sparse ROI-heavy: ~1-2% of pixels change


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_config_shapes(name):
    c = synth.get_config(name)
    assert c.n_bins == {"C1": 11, "C2": 101, "C3": 201, "C4": 401, "C5": 1001}[name]
    g = synth.geometry(c)
    assert g["wire_xyz"].shape == (c.n_steps, 3)
    assert oracle.Geometry(g).n_bins == c.n_bins


def test_travel_sweeps_bins_at_every_corner_pixel():
    """Every pixel's depth sweep covers [lo_0 - margin, hi_{M-1} + margin] (needed by the
    conservation-style parity checks and by the contributing-fraction estimate)."""
    for name in ("C1", "C2", "C4"):
        c = synth.get_config(name)
        g = synth.geometry(c)
        W = g["wire_xyz"]
        lo0 = c.depth_start - c.depth_res / 2
        hi = c.depth_end + c.depth_res / 2
        axis = np.array(g["wire_axis"])
        for (x, j) in [(-0.5, 0), (c.n - 0.5, 0), (-0.5, c.n - 1), (c.n - 0.5, c.n - 1)]:
            Q = oracle.detector_point(g, x, j)
            for edge in c.edges:
                s = oracle.edge_sigma(Q, W[0], W[-1], axis, edge)
                d0 = oracle.tangent_depth(Q, W[0], axis, g["wire_radius"], s, g["beam_dir"], g["beam_origin"])
                d1 = oracle.tangent_depth(Q, W[-1], axis, g["wire_radius"], s, g["beam_dir"], g["beam_origin"])
                assert min(d0, d1) < lo0 - 2 and max(d0, d1) > hi + 2, (name, x, j, edge, d0, d1)


def test_crop_geometry_keeps_pixel_positions():
    """A cropped detector's pixel (j, i) sits where the full detector's (row0 + j, col0 + i) does."""
    import indep
    g = synth.geometry("C5")
    c = synth.crop_geometry("C5", 1000, 1792, 64, 128)
    for (j, i) in [(0, 0), (63, 127), (10, 77)]:
        a = indep.detector_xyz(c, i, j)
        b = indep.detector_xyz(g, 1792 + i, 1000 + j)
        assert np.allclose(a, b, rtol=0, atol=1e-6)
