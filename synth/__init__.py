"""Seeded synthetic inputs for the DAXM wire-scan depth reconstruction.

This module is shared by BOTH the oracle tests and the CUDA path, so it holds
none of the method's arithmetic (no tangent ray-trace, no trapezoid, no
deposit).  It only produces *inputs*:

* the five workload configurations of ``BASELINE.json`` (``configs[0..4]``,
  called C1..C5 here, dimensions per SURVEY.md §8(d));
* a 34-ID-E-like geometry (detector pitch/rotation/translation, beam, wire
  axis/radius and the per-step wire-centre positions W_k), SURVEY.md §8(d)
  "Synthetic geometry".  W_k is a straight line, W(t) = W0 + t*d;
* an image stack I[k][row][col] built in *integer* arithmetic from a few
  per-pixel integer maps, so numpy (CPU, for the oracle) and torch (GPU, for
  the kernels) produce bit-identical values.

Stack recipe: background counts (1000 + a smooth
gradient, step independent, so dI = 0 there) plus single-grain Laue peaks
(2-D Gaussians, log-uniform amplitudes).  A peak pixel is dimmed while the
wire's leading edge crosses the grain slab and brightened back when the
trailing edge crosses it.  The step interval of that crossing comes from a
crude per-column *linear* fit (t0 + z * dt/dz, numbers below) - deliberately
not the method's ray-trace; it only has to put the change near the slab.
Optional counter-based integer noise makes every (pixel, step) non-constant,
which the parity tests use to exercise every output bin.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 220113309  # config seed = base + config number

# Wire travel t (um) along d = (0,1,1)/sqrt2, identical for every config, so
# only the step size changes with S.  [40, 880] sweeps [-55, +55] um of depth at
# every pixel of the 409.6 mm detector (checked by tests/test_synth.py
# through the oracle).
T_FIRST_UM = 40.0
T_LAST_UM = 880.0
T_LAST_TRAIL_UM = 1040.0  # the trailing edge lags one wire diameter: C2 scans further
WIRE_OFFSET_UM = 300.0  # W0 = 300 * (0,1,-1)/sqrt2 (300 um off a 45-degree surface)
WIRE_RADIUS_UM = 26.0
DET_SIZE_UM = 409600.0
DET_ROT = (-1.20161, -1.21837, -1.21741)  # ~0.7 deg off -120 deg about (1,1,1)
DET_TRANS = (25280.0, -2080.0, 510990.0)

# Crude linear occlusion model for the generator only (col 0 -> col C-1):
# the leading edge crosses depth z at t = t0 + z * inv_slope.  The end-point
# values were read off once from a plot of the geometry; they are inputs, not
# a claim about the method.
_T0_COL0, _T0_COLN = 113.8, 711.3
_INV_SLOPE_COL0, _INV_SLOPE_COLN = 1.0 / 0.959, 1.0 / 0.392
_TRAIL_SHIFT_UM = 2.0 * WIRE_RADIUS_UM * math.sqrt(2.0)  # wire diameter along d

FRAC_BITS = 10  # step positions in the integer recipe are in 1/1024 step


@dataclass(frozen=True)
class Config:
    name: str
    number: int
    n: int  # detector is n x n
    n_steps: int
    depth_res: float
    dtype: str  # "f32" | "u16"
    edges: tuple = ("leading",)
    sparse: bool = False
    n_peaks: int = 0
    depth_start: float = -50.0
    depth_end: float = 50.0
    slabs: tuple = ((-12.0, 9.0),)
    description: str = ""
    t_range: tuple = (T_FIRST_UM, T_LAST_UM)  # wire travel (um); C2 also covers the trailing edge

    @property
    def n_bins(self) -> int:
        return int(round((self.depth_end - self.depth_start) / self.depth_res)) + 1

    @property
    def seed(self) -> int:
        return SEED_BASE + self.number

    @property
    def pitch(self) -> float:
        return DET_SIZE_UM / self.n


CONFIGS = {
    "C1": Config("C1", 1, 64, 21, 10.0, "f32", ("leading",), False, 3,
                 description="64x64 detector, 21 wire steps, 11 depth bins, leading edge"),
    "C2": Config("C2", 2, 512, 201, 1.0, "f32", ("leading", "trailing"), False, 8,
                 t_range=(T_FIRST_UM, T_LAST_TRAIL_UM),
                 description="512x512, 201 steps, 101 bins at 1 um, leading and trailing"),
    "C3": Config("C3", 3, 1024, 401, 0.5, "u16", ("leading",), False, 30,
                 description="1024x1024, 401 steps, 201 bins at 0.5 um, uint16"),
    "C4": Config("C4", 4, 2048, 801, 0.25, "u16", ("leading",), False, 120,
                 description="2048x2048 PerkinElmer-style, 801 steps, 401 bins"),
    "C5": Config("C5", 5, 2048, 1601, 0.1, "u16", ("leading",), True, 1200,
                 slabs=((-30.0, -22.0), (-5.0, 3.0), (18.0, 27.0)),
                 description="2048x2048, 1601 fine steps, 1001 bins at 0.1 um, sparse ROIs"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name.upper()]


def wire_travel(n_steps: int, t_range: tuple = (T_FIRST_UM, T_LAST_UM)) -> np.ndarray:
    """t_k (um) for k = 0..S-1, uniform on t_range."""
    t0, t1 = t_range
    return t0 + (t1 - t0) * np.arange(n_steps, dtype=np.float64) / (n_steps - 1)


def wire_positions(n_steps: int, t: np.ndarray | None = None, t_range: tuple = (T_FIRST_UM, T_LAST_UM)) -> np.ndarray:
    """W_k = W0 + t_k * d, lab frame um, shape [S, 3] float64."""
    if t is None:
        t = wire_travel(n_steps, t_range)
    s2 = math.sqrt(2.0)
    w0 = np.array([0.0, WIRE_OFFSET_UM / s2, -WIRE_OFFSET_UM / s2])
    d = np.array([0.0, 1.0 / s2, 1.0 / s2])
    return w0[None, :] + t[:, None] * d[None, :]


def jittered_wire_positions(n_steps: int, t_range: tuple = (T_FIRST_UM, T_LAST_UM), amp_um: float = 0.3,
                            seed: int = 2201) -> np.ndarray:
    """A non-straight scan: the straight positions plus seeded jitter of up
    to +-amp_um perpendicular to both the scan line and the wire axis, and along the axis."""
    w = wire_positions(n_steps, t_range=t_range)
    rng = np.random.default_rng(seed)
    s2 = math.sqrt(2.0)
    perp = np.array([0.0, 1.0 / s2, -1.0 / s2])
    w = w + rng.uniform(-amp_um, amp_um, n_steps)[:, None] * perp[None, :]
    w[:, 0] += rng.uniform(-amp_um, amp_um, n_steps)
    return w


def geometry(cfg: Config | str, edge: str = "leading", pixel_model: str = "finite",
             n_rows: int | None = None, n_cols: int | None = None) -> dict:
    """Plain-number geometry dict consumed by both sides (each fills its own struct)."""
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    return dict(
        n_rows=n_rows or cfg.n, n_cols=n_cols or cfg.n,
        pitch_col=cfg.pitch, pitch_row=cfg.pitch,
        det_rot=DET_ROT, det_trans=DET_TRANS,
        beam_dir=(0.0, 0.0, 1.0), beam_origin=(0.0, 0.0, 0.0),
        wire_axis=(1.0, 0.0, 0.0), wire_radius=WIRE_RADIUS_UM,
        wire_xyz=wire_positions(cfg.n_steps, t_range=cfg.t_range),
        depth_start=cfg.depth_start, depth_end=cfg.depth_end, depth_res=cfg.depth_res,
        edge=edge, pixel_model=pixel_model,
    )


def crop_geometry(cfg: Config | str, row0: int, col0: int, n_rows: int, n_cols: int, **kw) -> dict:
    """The geometry of the detector window rows [row0, row0 + n_rows) x columns [col0, col0 + n_cols)
    of `cfg`'s detector: the same pixels, in the same lab positions (det_trans shifted in the
    detector plane by the window centre's offset), so a small test sees the depth spans and
    step spacings of any region of a full-size configuration."""
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    g = geometry(cfg, n_rows=n_rows, n_cols=n_cols, **kw)
    dx = (col0 + (n_cols - 1) / 2.0 - (cfg.n - 1) / 2.0) * cfg.pitch
    dy = (row0 + (n_rows - 1) / 2.0 - (cfg.n - 1) / 2.0) * cfg.pitch
    g["det_trans"] = (DET_TRANS[0] + dx, DET_TRANS[1] + dy, DET_TRANS[2])
    return g


# ----------------------------------------------------------------------------
# Integer stack recipe
# ----------------------------------------------------------------------------

@dataclass
class StackMaps:
    """Per-pixel integer maps; I[k] = bg + noise + amp - lead(k) + trail(k)."""
    n_rows: int
    n_cols: int
    n_steps: int
    bg: np.ndarray     # int64 [R, C]
    amp: np.ndarray    # int64 [R, C]
    ka: np.ndarray     # int64 [R, C], leading-crossing start, 1/1024 step units
    w: np.ndarray      # int64 [R, C], crossing width (>= 1), same units
    kt: np.ndarray     # int64 [R, C], trailing-crossing start
    seed: int = 0
    meta: dict = field(default_factory=dict)


def make_maps(cfg: Config | str, n_peaks: int | None = None, seed: int | None = None) -> StackMaps:
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    R = C = cfg.n
    S = cfg.n_steps
    seed = cfg.seed if seed is None else seed
    rng = np.random.default_rng(seed)
    n_peaks = cfg.n_peaks if n_peaks is None else n_peaks

    jj, ii = np.meshgrid(np.arange(R, dtype=np.float64), np.arange(C, dtype=np.float64), indexing="ij")
    bg = (1000.0 + 200.0 * ii / max(C - 1, 1) + 100.0 * jj / max(R - 1, 1)).round().astype(np.int64)

    sigma = max(0.7, 1.5 * 200.0 / cfg.pitch)
    half = 3 if cfg.sparse else int(math.ceil(4.0 * sigma))  # 7x7 ROI in the sparse config
    amp_f = np.zeros((R, C), dtype=np.float64)
    grain = np.full((R, C), -1, dtype=np.int64)
    best = np.zeros((R, C), dtype=np.float64)
    py = rng.uniform(half, R - 1 - half, n_peaks)
    px = rng.uniform(half, C - 1 - half, n_peaks)
    logA = rng.uniform(math.log(200.0), math.log(20000.0), n_peaks)
    g_of = rng.integers(0, len(cfg.slabs), n_peaks)
    for p in range(n_peaks):
        cy, cx = int(round(py[p])), int(round(px[p]))
        y0, y1 = max(cy - half, 0), min(cy + half + 1, R)
        x0, x1 = max(cx - half, 0), min(cx + half + 1, C)
        yy, xx = np.meshgrid(np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
        g = math.exp(logA[p]) * np.exp(-((yy - py[p]) ** 2 + (xx - px[p]) ** 2) / (2 * sigma * sigma))
        amp_f[y0:y1, x0:x1] += g
        upd = g > best[y0:y1, x0:x1]
        best[y0:y1, x0:x1] = np.where(upd, g, best[y0:y1, x0:x1])
        grain[y0:y1, x0:x1] = np.where(upd, g_of[p], grain[y0:y1, x0:x1])
    amp = np.minimum(amp_f.round(), 60000.0).astype(np.int64)
    amp[amp < 1] = 0

    # crude per-column linear occlusion model -> step interval (generator only)
    xi = ii / max(C - 1, 1)
    t0 = _T0_COL0 + (_T0_COLN - _T0_COL0) * xi
    inv_slope = _INV_SLOPE_COL0 + (_INV_SLOPE_COLN - _INV_SLOPE_COL0) * xi
    slabs = np.array(cfg.slabs, dtype=np.float64)
    gsel = np.maximum(grain, 0)
    za, zb = slabs[gsel, 0], slabs[gsel, 1]
    steps_per_um = (S - 1) / (cfg.t_range[1] - cfg.t_range[0])
    k_a = (t0 + za * inv_slope - cfg.t_range[0]) * steps_per_um
    k_b = (t0 + zb * inv_slope - cfg.t_range[0]) * steps_per_um
    scale = float(1 << FRAC_BITS)
    ka = np.round(k_a * scale).astype(np.int64)
    w = np.maximum(np.round((k_b - k_a) * scale).astype(np.int64), 1)
    kt = ka + np.round(_TRAIL_SHIFT_UM * steps_per_um * scale).astype(np.int64)
    return StackMaps(R, C, S, bg, amp, ka, w, kt, seed,
                     meta=dict(sigma_px=sigma, n_peaks=n_peaks, config=cfg.name))


def _mix(k, j, i, seed, xp):
    """Counter-based integer hash of (seed, k, row, col) -> [0, 2^31)."""
    m = 0x7FFFFFFF
    h = ((k * 73856093) ^ (j * 19349663) ^ (i * 83492791) ^ seed) & m
    h = (h * 1103515245 + 12345) & m
    h = (h ^ (h >> 13)) & m
    h = (h * 1103515245 + 12345) & m
    return h


def stack_values(k, j, i, bg, amp, ka, w, kt, seed, noise, xp):
    """Integer stack value I[k][j][i] (int64), element-wise; xp = numpy or torch.

    All operands broadcast; only integer +,-,*,//,&,^,>>, min/max are used so
    numpy and torch agree bit for bit.
    """
    num = k * (1 << FRAC_BITS)
    lead = (amp * xp.clip(num - ka, 0, None).clip(None, w)) // w if xp is np else \
        (amp * (num - ka).clamp(min=0).minimum(w)) // w
    trail = (amp * xp.clip(num - kt, 0, None).clip(None, w)) // w if xp is np else \
        (amp * (num - kt).clamp(min=0).minimum(w)) // w
    val = bg + amp - lead + trail
    if noise:
        h = _mix(k, j, i, seed, xp)
        val = val + (h >> 16) % 17 - 8
    return val


def to_dtype(vals, dtype: str, xp):
    if dtype == "u16":
        v = vals.clip(0, 65535) if xp is np else vals.clamp(0, 65535)
        return v.astype(np.uint16) if xp is np else v.to(xp.uint16)
    if dtype == "f32":
        return vals.astype(np.float32) if xp is np else vals.to(xp.float32)
    if dtype == "f64":
        return vals.astype(np.float64) if xp is np else vals.to(xp.float64)
    raise ValueError(dtype)


def stack_numpy(maps: StackMaps, dtype: str, noise: bool = False, rows: tuple | None = None) -> np.ndarray:
    """Full (or row-band) stack [S][rows][C] on the host."""
    r0, r1 = rows or (0, maps.n_rows)
    sl = slice(r0, r1)
    jj, ii = np.meshgrid(np.arange(r0, r1, dtype=np.int64), np.arange(maps.n_cols, dtype=np.int64), indexing="ij")
    out = np.empty((maps.n_steps, r1 - r0, maps.n_cols), dtype={"u16": np.uint16, "f32": np.float32, "f64": np.float64}[dtype])
    for k in range(maps.n_steps):
        v = stack_values(np.int64(k), jj, ii, maps.bg[sl], maps.amp[sl], maps.ka[sl], maps.w[sl], maps.kt[sl],
                         maps.seed, noise, np)
        out[k] = to_dtype(v, dtype, np)
    return out


def pixel_series(maps: StackMaps, js, is_, dtype: str, noise: bool = False) -> np.ndarray:
    """I[:, j, i] for a list of pixels -> [n, S] (host), identical to the full stack."""
    js = np.asarray(js, dtype=np.int64)
    is_ = np.asarray(is_, dtype=np.int64)
    k = np.arange(maps.n_steps, dtype=np.int64)[None, :]
    j, i = js[:, None], is_[:, None]
    v = stack_values(k, j, i, maps.bg[js, is_][:, None], maps.amp[js, is_][:, None], maps.ka[js, is_][:, None],
                     maps.w[js, is_][:, None], maps.kt[js, is_][:, None], maps.seed, noise, np)
    return to_dtype(v, dtype, np)


def stack_torch(maps: StackMaps, dtype: str, device, noise: bool = False, rows: tuple | None = None, out=None):
    """Full (or row-band) stack [S][rows][C] generated on `device` (outside any timed region)."""
    import torch
    r0, r1 = rows or (0, maps.n_rows)
    tdt = {"u16": torch.uint16, "f32": torch.float32, "f64": torch.float64}[dtype]
    if out is None:
        out = torch.empty((maps.n_steps, r1 - r0, maps.n_cols), dtype=tdt, device=device)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a[r0:r1])).to(device)
    bg, amp, ka, w, kt = dev(maps.bg), dev(maps.amp), dev(maps.ka), dev(maps.w), dev(maps.kt)
    jj = torch.arange(r0, r1, device=device, dtype=torch.int64)[None, :, None]
    ii = torch.arange(maps.n_cols, device=device, dtype=torch.int64)[None, None, :]
    bg, amp, ka, w, kt = (x[None] for x in (bg, amp, ka, w, kt))
    # a few steps per launch group (bounded temporary memory: int64 [kc, rows, C])
    kc = max(1, min(maps.n_steps, (1 << 28) // max(1, (r1 - r0) * maps.n_cols)))
    for k0 in range(0, maps.n_steps, kc):
        k1 = min(maps.n_steps, k0 + kc)
        k = torch.arange(k0, k1, device=device, dtype=torch.int64)[:, None, None]
        v = stack_values(k, jj, ii, bg, amp, ka, w, kt, maps.seed, noise, torch)
        out[k0:k1].copy_(to_dtype(v, dtype, torch))
    return out
