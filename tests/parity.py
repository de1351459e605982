"""Parity tolerance of BASELINE.json north_star, written out once.

per bin:   |gpu - oracle| <= 1e-4 * sum_k |dI_k(p)|
per pixel: |sum_m gpu - sum_m oracle| <= 1e-5 * max(|sum_m oracle|, sum_k |dI_k(p)|)
(the max() denominator is SURVEY.md §8(c)'s reading for background pixels whose
sum is ~0).  Arrays are [M, ...pixels] (output) and [S, ...pixels] (stack).
"""
import numpy as np

BIN_TOL = 1e-4
SUM_TOL = 1e-5


def abs_dI(series: np.ndarray) -> np.ndarray:
    s = np.asarray(series, dtype=np.float64)
    return np.abs(np.diff(s, axis=0)).sum(0)


def check(gpu, ref, series, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    assert np.isfinite(gpu).all(), f"{what}: non-finite GPU output"
    d = abs_dI(series)
    err = np.abs(gpu - ref)
    lim = np.broadcast_to(BIN_TOL * d[None], err.shape)
    bad = err > lim
    if bad.any():
        idx = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} bins over tolerance; first {tuple(idx)}: gpu {gpu[tuple(idx)]}"
                             f" oracle {ref[tuple(idx)]} tol {lim[tuple(idx)]}; max err/sum|dI| "
                             f"{(err / np.maximum(d[None], 1e-300)).max():.3g}")
    sg, sr = gpu.sum(0), ref.sum(0)
    slim = SUM_TOL * np.maximum(np.abs(sr), d)
    sbad = np.abs(sg - sr) > slim
    if sbad.any():
        idx = np.argwhere(sbad)[0]
        raise AssertionError(f"{what}: {int(sbad.sum())} pixel sums over tolerance; first {tuple(idx)}: "
                             f"{sg[tuple(idx)]} vs {sr[tuple(idx)]}")
    rel = err / np.maximum(d[None], 1e-300)
    return float(np.where(d[None] > 0, rel, 0).max())
