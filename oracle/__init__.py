"""ctypes binding of the fp64 CPU oracle (oracle/daxm_oracle.c).

TEST INFRASTRUCTURE ONLY -- only tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py may import this module.
It shares no code with the CUDA path (paper_2201_13309_b200/) and never
imports it.  See daxm_oracle.c for the paper citations of each step.

Parity status of each exported function:
  oracle_rodrigues, oracle_detector_point      pinned (tests/test_oracle_geometry.py)
  oracle_tangent_depth, oracle_edge_sigma      pinned (closed form, special case, r->0, invariances)
  oracle_trapezoid_cdf, oracle_deposit_pair    pinned (numeric integration, box overlap, brute force)
  oracle_reconstruct[_pixels]                  pinned (conservation, background, linearity,
                                               reversal identity, forward-model round trip)
  select_cutoff, active_pixels (python)        pinned (order-statistic definition, tests/test_oracle_cutoff.py)
  edge "both" (reading R16)                    pinned (tests/test_oracle_both.py: split identity
                                               both(I) = lead(D) + trail(U) through the pinned single-edge
                                               oracle, monotone stacks, forward-model point scatterer)
  depth_profile (python)                       pinned (conservation: the profile's total = sum_p s (I_0 - I_{S-1})
                                               when every trapezoid lies inside the bins; a single non-constant
                                               pixel's profile = its oracle_reconstruct_pixels column;
                                               tests/test_oracle_cutoff.py)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "daxm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


class OracleGeometry(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_cols", C.c_int32),
        ("pitch_col", C.c_double), ("pitch_row", C.c_double),
        ("det_rot", C.c_double * 3), ("det_trans", C.c_double * 3),
        ("beam_dir", C.c_double * 3), ("beam_origin", C.c_double * 3),
        ("wire_axis", C.c_double * 3), ("wire_radius", C.c_double),
        ("n_steps", C.c_int32), ("wire_xyz", C.POINTER(C.c_double)),
        ("depth_start", C.c_double), ("depth_end", C.c_double), ("depth_res", C.c_double),
        ("edge", C.c_int32), ("pixel_model", C.c_int32), ("raw_sign", C.c_int32),
        ("step_weight", C.POINTER(C.c_double)),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (plain -O2, IEEE fp64, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        L.oracle_rodrigues.argtypes = [dp, dp]
        L.oracle_detector_point.argtypes = [C.POINTER(OracleGeometry), C.c_double, C.c_double, dp]
        L.oracle_tangent_depth.argtypes = [dp, dp, dp, C.c_double, C.c_double, dp, dp]
        L.oracle_tangent_depth.restype = C.c_double
        L.oracle_edge_sigma.argtypes = [dp, dp, dp, dp, C.c_int]
        L.oracle_edge_sigma.restype = C.c_double
        L.oracle_trapezoid_cdf.argtypes = [dp, C.c_double]
        L.oracle_trapezoid_cdf.restype = C.c_double
        L.oracle_deposit_pair.argtypes = [C.c_double, dp, C.c_double, C.c_double, C.c_int, dp, C.c_long]
        L.oracle_n_bins.argtypes = [C.POINTER(OracleGeometry)]
        L.oracle_reconstruct_pixels.argtypes = [C.POINTER(OracleGeometry), C.c_int, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_int32), dp, dp, C.c_int]
        L.oracle_reconstruct.argtypes = [C.POINTER(OracleGeometry), C.c_void_p, C.c_int, dp, C.c_int, C.c_int,
                                         C.c_int]
        L.oracle_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _v3(x):
    return (C.c_double * 3)(*[float(v) for v in x])


class Geometry:
    """Holds an OracleGeometry plus the arrays it points to."""

    def __init__(self, g: dict, raw_sign: bool = False):
        self.wire = np.ascontiguousarray(np.asarray(g["wire_xyz"], dtype=np.float64).reshape(-1, 3))
        edge = {"leading": 0, "trailing": 1, "both": 2}[g.get("edge", "leading")]
        pm = {"finite": 0, "point": 1}[g.get("pixel_model", "finite")]
        self.s = OracleGeometry(
            int(g["n_rows"]), int(g["n_cols"]), float(g["pitch_col"]), float(g["pitch_row"]),
            _v3(g["det_rot"]), _v3(g["det_trans"]), _v3(g["beam_dir"]), _v3(g["beam_origin"]),
            _v3(g["wire_axis"]), float(g["wire_radius"]), int(self.wire.shape[0]), _dp(self.wire),
            float(g["depth_start"]), float(g["depth_end"]), float(g["depth_res"]), edge, pm, int(raw_sign),
            None)
        w = g.get("step_weight")
        if w is not None:  # per-step intensity normalisation (reading R17)
            self.weight = np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(-1))
            assert self.weight.shape[0] == self.wire.shape[0]
            self.s.step_weight = _dp(self.weight)

    @property
    def n_bins(self) -> int:
        return lib().oracle_n_bins(C.byref(self.s))


def rodrigues(R) -> np.ndarray:
    R = np.ascontiguousarray(R, dtype=np.float64)
    out = np.zeros(9)
    lib().oracle_rodrigues(_dp(R), _dp(out))
    return out.reshape(3, 3)


def detector_point(g: dict, x: float, j: float) -> np.ndarray:
    G = Geometry(g)
    out = np.zeros(3)
    lib().oracle_detector_point(C.byref(G.s), float(x), float(j), _dp(out))
    return out


def tangent_depth(Q, W, axis, r, sigma, beam=(0, 0, 1), origin=(0, 0, 0)) -> float:
    a = [np.ascontiguousarray(v, dtype=np.float64) for v in (Q, W, axis, beam, origin)]
    return lib().oracle_tangent_depth(_dp(a[0]), _dp(a[1]), _dp(a[2]), float(r), float(sigma), _dp(a[3]),
                                      _dp(a[4]))


def edge_sigma(Q, W0, Wlast, axis, edge: str = "leading") -> float:
    a = [np.ascontiguousarray(v, dtype=np.float64) for v in (Q, W0, Wlast, axis)]
    return lib().oracle_edge_sigma(_dp(a[0]), _dp(a[1]), _dp(a[2]), _dp(a[3]), 0 if edge == "leading" else 1)


def trapezoid_cdf(z, x: float) -> float:
    z = np.ascontiguousarray(z, dtype=np.float64)
    return lib().oracle_trapezoid_cdf(_dp(z), float(x))


def deposit_pair(dI: float, corners, start: float, dz: float, M: int) -> np.ndarray:
    c = np.ascontiguousarray(corners, dtype=np.float64)
    out = np.zeros(M)
    lib().oracle_deposit_pair(float(dI), _dp(c), float(start), float(dz), int(M), _dp(out), 1)
    return out


def reconstruct_pixels(g: dict, rows, cols, series: np.ndarray, n_threads: int = 0,
                       raw_sign: bool = False) -> np.ndarray:
    """series [n, S] -> out [n, M] fp64."""
    G = Geometry(g, raw_sign=raw_sign)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    ser = np.ascontiguousarray(series, dtype=np.float64)
    n = rows.shape[0]
    assert ser.shape == (n, G.s.n_steps)
    out = np.zeros((n, G.n_bins))
    st = lib().oracle_reconstruct_pixels(C.byref(G.s), n, rows.ctypes.data_as(C.POINTER(C.c_int32)),
                                         cols.ctypes.data_as(C.POINTER(C.c_int32)), _dp(ser), _dp(out),
                                         int(n_threads))
    if st != 0:
        raise ValueError("oracle_reconstruct_pixels: invalid argument")
    return out


def reconstruct(g: dict, stack: np.ndarray, rows: tuple | None = None, n_threads: int = 0,
                raw_sign: bool = False) -> np.ndarray:
    """stack [S][R][C] (uint16 / float32 / float64) -> out [M][R][C] fp64 (rows outside band = 0)."""
    G = Geometry(g, raw_sign=raw_sign)
    stack = np.ascontiguousarray(stack)
    dt = {np.dtype(np.uint16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}[stack.dtype]
    S, R, Cc = stack.shape
    assert (S, R, Cc) == (G.s.n_steps, G.s.n_rows, G.s.n_cols), (stack.shape, G.s.n_steps)
    r0, r1 = rows or (0, R)
    out = np.zeros((G.n_bins, R, Cc))
    st = lib().oracle_reconstruct(C.byref(G.s), stack.ctypes.data_as(C.c_void_p), dt, _dp(out), r0, r1,
                                  int(n_threads))
    if st != 0:
        raise ValueError("oracle_reconstruct: invalid argument")
    return out


def active_pixels(first_image: np.ndarray, cutoff: float) -> np.ndarray:
    """Intensity cutoff (d_cutoff; reading R14): a pixel is processed iff its
    first wire-step intensity I_0, compared in float32, is >= cutoff."""
    return np.asarray(first_image).astype(np.float32) >= np.float32(cutoff)


def select_cutoff(first_image: np.ndarray, fraction: float) -> float:
    """Pixel percentage (reading R14): the k-th largest I_0, k = ceil(fraction * n)
    clamped to [1, n]; NaN ranks lowest.  Plain sort."""
    import math
    v = np.asarray(first_image, dtype=np.float64).ravel()
    n = v.size
    k = min(max(int(math.ceil(fraction * n)), 1), n)
    v = np.where(np.isnan(v), -np.inf, v)
    return float(np.sort(v)[::-1][k - 1])


def reconstruct_cutoff(g: dict, stack: np.ndarray, cutoff: float, rows: tuple | None = None,
                       n_threads: int = 0) -> np.ndarray:
    """reconstruct() with the intensity cutoff: pixels below it are not processed (output 0)."""
    out = reconstruct(g, stack, rows=rows, n_threads=n_threads)
    out[:, ~active_pixels(np.asarray(stack)[0], cutoff)] = 0.0
    return out


def depth_profile(out: np.ndarray) -> np.ndarray:
    """image_set.depth_intensity: per-bin total over all pixels, fp64."""
    return np.asarray(out, dtype=np.float64).sum(axis=(1, 2))


def max_threads() -> int:
    return lib().oracle_max_threads()
