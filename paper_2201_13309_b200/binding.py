"""ctypes binding of libdaxm.so (include/daxm.h) -- argument marshalling only.

Names follow the C ABI: ``create`` -> daxm_create, ``Plan.reconstruct`` ->
daxm_reconstruct (device tensors, torch's current stream),
``Plan.reconstruct_host`` -> daxm_reconstruct_host (host arrays).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# DAXM_LIBRARY selects an alternative build of the same library (kernel-variant experiments)
_LIB_PATH = os.environ.get("DAXM_LIBRARY") or os.path.join(_PKG, "libdaxm.so")

EDGE = {"leading": 0, "trailing": 1, "both": 2}
PIXEL_MODEL = {"finite": 0, "point": 1}
DTYPE = {"u16": 0, "f32": 1}

STATUS = {0: "ok", 1: "invalid argument", 2: "non-monotone scan", 3: "geometry error", 4: "out of memory",
          5: "CUDA error"}


class DaxmError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


class Geometry(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32),
        ("pitch_col", C.c_double), ("pitch_row", C.c_double),
        ("det_rot", C.c_double * 3), ("det_trans", C.c_double * 3),
        ("beam_dir", C.c_double * 3), ("beam_origin", C.c_double * 3),
        ("wire_axis", C.c_double * 3), ("wire_radius", C.c_double),
        ("n_steps", C.c_int32), ("wire_xyz", C.POINTER(C.c_double)),
        ("depth_start", C.c_double), ("depth_end", C.c_double), ("depth_res", C.c_double),
        ("edge", C.c_int32), ("pixel_model", C.c_int32),
    ]


# daxm_hist_reduce_fn (include/daxm.h): int (*)(unsigned long long *hist, int n, void *ctx)
HIST_REDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_ulonglong), C.c_int, C.c_void_p)


class PlanStats(C.Structure):
    _fields_ = [
        ("n_bins", C.c_int64), ("rows", C.c_int64), ("cols", C.c_int64), ("n_steps", C.c_int64),
        ("contrib_pairs", C.c_int64), ("contrib_pixels", C.c_int64), ("window_pairs", C.c_int64), ("staged_steps", C.c_int64), ("n_tiles", C.c_int64),
        ("general_tiles_u16", C.c_int64), ("general_tiles_f32", C.c_int64),
        ("nonseparated_tiles", C.c_int64), ("overlap_tiles", C.c_int64), ("ring_need_max", C.c_int64),
        ("tile_rows", C.c_int32), ("tile_cols", C.c_int32),
        ("fit_max_err_bins", C.c_double), ("fit_model_err_bins", C.c_double), ("prepass_ms", C.c_double), ("device_bytes", C.c_int64),
        ("depth_table_bytes", C.c_int64),
        ("lock_tiles_small", C.c_int64), ("lock_tiles_large", C.c_int64), ("lock_ring_violations", C.c_int64),
        ("lock_tiles_overlap", C.c_int64),
        ("row_tiles_small", C.c_int64), ("row_tiles_large", C.c_int64), ("row_tiles_general", C.c_int64),
        ("row_ring_need_max", C.c_int64), ("row_reject_bits", C.c_int64), ("row_reject", C.c_int64 * 8),
        ("row_path", C.c_int64), ("row_tiles_gen", C.c_int64), ("row_reject_more", C.c_int64),
        ("row_launches", C.c_int64), ("row_tiles_nb_mid", C.c_int64), ("row_kmax_hist", C.c_int64 * 8),
    ]


_lib = None


def lib():
    """Load libdaxm.so (fails loudly if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        L.daxm_create.argtypes = [C.POINTER(Geometry), C.c_int, C.POINTER(P)]
        L.daxm_create.restype = C.c_int
        L.daxm_plan_info.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.daxm_plan_info.restype = C.c_int
        L.daxm_plan_stats_get.argtypes = [P, C.POINTER(PlanStats)]
        L.daxm_plan_stats_get.restype = C.c_int
        L.daxm_reconstruct.argtypes = [P, P, C.c_int, P, P]
        L.daxm_reconstruct.restype = C.c_int
        L.daxm_reconstruct_host.argtypes = [P, P, C.c_int, P, P]
        L.daxm_reconstruct_host.restype = C.c_int
        # (newer entry points: a build of an older source, DAXM_LIBRARY experiments, may lack them)
        if hasattr(L, "daxm_set_step_weights"):
            L.daxm_set_step_weights.argtypes = [P, C.POINTER(C.c_double)]
            L.daxm_set_step_weights.restype = C.c_int
        if hasattr(L, "daxm_set_host_budget"):
            L.daxm_set_host_budget.argtypes = [P, C.c_uint64]
            L.daxm_set_host_budget.restype = C.c_int
            L.daxm_host_ring_info.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.daxm_host_ring_info.restype = C.c_int
        L.daxm_set_cutoff.argtypes = [P, C.c_int, C.c_double]
        L.daxm_set_cutoff.restype = C.c_int
        L.daxm_select_cutoff.argtypes = [P, P, C.c_int, C.c_double, C.POINTER(C.c_double), P]
        L.daxm_select_cutoff.restype = C.c_int
        L.daxm_select_cutoff_sharded.argtypes = [P, P, C.c_int, C.c_double, C.c_ulonglong, HIST_REDUCE_FN, P,
                                                 C.POINTER(C.c_double), P]
        L.daxm_select_cutoff_sharded.restype = C.c_int
        L.daxm_depth_profile.argtypes = [P, P, P, P]
        L.daxm_depth_profile.restype = C.c_int
        L.daxm_reconstruct_profile.argtypes = [P, P, C.c_int, P, P, P]
        L.daxm_reconstruct_profile.restype = C.c_int
        L.daxm_last_error.argtypes = [P]
        L.daxm_last_error.restype = C.c_char_p
        L.daxm_create_error.restype = C.c_char_p
        L.daxm_status_string.argtypes = [C.c_int]
        L.daxm_status_string.restype = C.c_char_p
        L.daxm_destroy.argtypes = [P]
        L.daxm_destroy.restype = None
        L.daxm_abi_version.restype = C.c_int
        _lib = L
    return _lib


def abi_version() -> int:
    return lib().daxm_abi_version()


def _v3(x):
    return (C.c_double * 3)(*[float(v) for v in x])


def make_geometry(g: dict, rows: tuple | None = None):
    """dict (synth.geometry format) -> (Geometry struct, keep-alive array)."""
    wire = np.ascontiguousarray(np.asarray(g["wire_xyz"], dtype=np.float64).reshape(-1, 3))
    r0, r1 = rows if rows is not None else (0, int(g["n_rows"]))
    s = Geometry(int(g["n_rows"]), int(g["n_cols"]), int(r0), int(r1), float(g["pitch_col"]), float(g["pitch_row"]),
                 _v3(g["det_rot"]), _v3(g["det_trans"]), _v3(g["beam_dir"]), _v3(g["beam_origin"]),
                 _v3(g["wire_axis"]), float(g["wire_radius"]), int(wire.shape[0]),
                 wire.ctypes.data_as(C.POINTER(C.c_double)), float(g["depth_start"]), float(g["depth_end"]),
                 float(g["depth_res"]), EDGE.get(g.get("edge", "leading"), g.get("edge")),
                 PIXEL_MODEL.get(g.get("pixel_model", "finite"), g.get("pixel_model")))
    return s, wire


class Plan:
    """Owns a daxm_plan*.  Use ``create(geometry_dict, device, rows)``."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device
        M, R, Cc = C.c_int64(), C.c_int64(), C.c_int64()
        lib().daxm_plan_info(self._h, C.byref(M), C.byref(R), C.byref(Cc))
        self.n_bins, self.rows, self.cols = M.value, R.value, Cc.value
        self.n_steps = self.stats()["n_steps"]

    def stack_shape(self):
        return (self.n_steps, self.rows, self.cols)

    def _check(self, st: int):
        if st != 0:
            raise DaxmError(st, lib().daxm_last_error(self._h).decode())

    def stats(self) -> dict:
        s = PlanStats()
        self._check(lib().daxm_plan_stats_get(self._h, C.byref(s)))
        return {f: (list(getattr(s, f)) if isinstance(getattr(s, f), C.Array) else getattr(s, f))
                for f, _ in PlanStats._fields_}

    def output_shape(self):
        return (self.n_bins, self.rows, self.cols)

    def reconstruct(self, stack, out=None, stream=None):
        """stack: CUDA tensor [S][rows][C] uint16 or float32 -> out [M][rows][C] float32 (CUDA)."""
        import torch
        dt = self._dtype_of(stack)
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=stack.device)
        if not (out.is_cuda and out.is_contiguous() and out.dtype == torch.float32 and
                tuple(out.shape) == self.output_shape() and out.device == stack.device):
            raise ValueError("out must be a contiguous float32 CUDA tensor of shape [M][rows][C] on the "
                             "stack's device")
        if stream is None:
            stream = torch.cuda.current_stream(stack.device)
        self._check(lib().daxm_reconstruct(self._h, C.c_void_p(stack.data_ptr()), dt, C.c_void_p(out.data_ptr()),
                                           C.c_void_p(stream.cuda_stream)))
        return out

    def _dtype_of(self, stack, plane0_only=False):
        """Validate a device stack (shape [S][rows][C] -- or at least its first plane --, contiguous,
        on the plan's device) and return its daxm_dtype."""
        import torch
        if not (stack.is_cuda and stack.is_contiguous()):
            raise ValueError("stack must be a contiguous CUDA tensor")
        if stack.device.index != self.device:
            raise ValueError(f"stack is on {stack.device}, the plan on cuda:{self.device}")
        shape = tuple(stack.shape)
        if plane0_only:
            ok = len(shape) == 3 and shape[1:] == self.stack_shape()[1:] and shape[0] >= 1
        else:
            ok = shape == self.stack_shape()
        if not ok:
            raise ValueError(f"stack shape {shape}, the plan needs {self.stack_shape()} [S][rows][C]")
        dt = {torch.uint16: 0, torch.float32: 1}.get(stack.dtype)
        if dt is None:
            raise ValueError(f"unsupported stack dtype {stack.dtype}")
        return dt

    def set_cutoff(self, cutoff):
        """Reconstruct only pixels with first-step intensity >= cutoff (None: all pixels)."""
        self._check(lib().daxm_set_cutoff(self._h, 0 if cutoff is None else 1,
                                          0.0 if cutoff is None else float(cutoff)))

    def select_cutoff(self, stack, fraction, stream=None):
        """The cutoff keeping `fraction` of the plan's pixels (k-th largest first-step intensity)."""
        import torch
        dt = self._dtype_of(stack, plane0_only=True)
        if stream is None:
            stream = torch.cuda.current_stream(stack.device)
        val = C.c_double()
        self._check(lib().daxm_select_cutoff(self._h, C.c_void_p(stack.data_ptr()), dt, float(fraction),
                                             C.byref(val), C.c_void_p(stream.cuda_stream)))
        return val.value

    def select_cutoff_sharded(self, stack, fraction, n_total, reduce, stream=None):
        """daxm_select_cutoff_sharded: the cutoff keeping `fraction` of `n_total` pixels split over
        row-band plans.  `reduce(hist)` sums a uint64 numpy array over the shards in place
        (multi.hist_allreduce builds one for torch.distributed)."""
        import numpy as np
        import torch
        dt = self._dtype_of(stack, plane0_only=True)
        if stream is None:
            stream = torch.cuda.current_stream(stack.device)
        errors = []

        def cb(hist, n, ctx):
            try:
                reduce(np.ctypeslib.as_array(hist, shape=(n,)))
                return 0
            except BaseException as e:  # reported after the C call returns
                errors.append(e)
                return 1
        fn = HIST_REDUCE_FN(cb)
        val = C.c_double()
        st = lib().daxm_select_cutoff_sharded(self._h, C.c_void_p(stack.data_ptr()), dt, float(fraction),
                                              int(n_total), fn, None, C.byref(val), C.c_void_p(stream.cuda_stream))
        if errors:
            raise errors[0]
        self._check(st)
        return val.value

    def reconstruct_profile(self, stack, out=None, profile=None, stream=None):
        """daxm_reconstruct_profile: reconstruction and its depth profile (fused on the row path)
        -> (out [M][rows][C] float32 CUDA, profile [M] float64 CUDA)."""
        import torch
        dt = self._dtype_of(stack)
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=stack.device)
        if not (out.is_cuda and out.is_contiguous() and out.dtype == torch.float32 and
                tuple(out.shape) == self.output_shape() and out.device == stack.device):
            raise ValueError("out must be a contiguous float32 CUDA tensor of shape [M][rows][C] on the "
                             "stack's device")
        if profile is None:
            profile = torch.empty(self.n_bins, dtype=torch.float64, device=stack.device)
        if not (profile.is_cuda and profile.is_contiguous() and profile.dtype == torch.float64 and
                tuple(profile.shape) == (self.n_bins,) and profile.device == stack.device):
            raise ValueError("profile must be a contiguous float64 CUDA tensor [M] on the stack's device")
        if stream is None:
            stream = torch.cuda.current_stream(stack.device)
        self._check(lib().daxm_reconstruct_profile(self._h, C.c_void_p(stack.data_ptr()), dt,
                                                   C.c_void_p(out.data_ptr()), C.c_void_p(profile.data_ptr()),
                                                   C.c_void_p(stream.cuda_stream)))
        return out, profile

    def depth_profile(self, out, profile=None, stream=None):
        """Per-depth-bin total intensity of `out` ([M][rows][C] float32 CUDA) -> float64 CUDA [M]."""
        import torch
        if not (out.is_cuda and out.is_contiguous() and out.dtype == torch.float32 and
                tuple(out.shape) == self.output_shape()):
            raise ValueError("out must be the plan's contiguous float32 CUDA output [M][rows][C]")
        if profile is None:
            profile = torch.empty(self.n_bins, dtype=torch.float64, device=out.device)
        if stream is None:
            stream = torch.cuda.current_stream(out.device)
        self._check(lib().daxm_depth_profile(self._h, C.c_void_p(out.data_ptr()), C.c_void_p(profile.data_ptr()),
                                             C.c_void_p(stream.cuda_stream)))
        return profile

    def reconstruct_host(self, stack, out=None, stream=None):
        """Host (numpy or pinned CPU torch) stack -> host output, copies included (daxm_reconstruct_host)."""
        import torch
        if isinstance(stack, np.ndarray):
            stack = torch.from_numpy(np.ascontiguousarray(stack))
        dt = {torch.uint16: 0, torch.float32: 1}.get(stack.dtype)
        if dt is None or stack.is_cuda or not stack.is_contiguous():
            raise ValueError("stack must be a contiguous host uint16/float32 tensor or array")
        if tuple(stack.shape) != self.stack_shape():
            raise ValueError(f"stack shape {tuple(stack.shape)}, the plan needs {self.stack_shape()} [S][rows][C]")
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, pin_memory=stack.is_pinned())
        elif isinstance(out, np.ndarray):
            if not (out.dtype == np.float32 and out.flags.c_contiguous and out.shape == self.output_shape()):
                raise ValueError("out must be a C-contiguous float32 array of shape [M][rows][C]")
            out = torch.from_numpy(out)
        elif not (not out.is_cuda and out.is_contiguous() and out.dtype == torch.float32 and
                  tuple(out.shape) == self.output_shape()):
            raise ValueError("out must be a contiguous float32 host tensor of shape [M][rows][C]")
        st = 0 if stream is None else stream.cuda_stream
        self._check(lib().daxm_reconstruct_host(self._h, C.c_void_p(stack.data_ptr()), dt,
                                                C.c_void_p(out.data_ptr()), C.c_void_p(st)))
        return out

    def set_step_weights(self, w):
        """Per-step intensity normalisation w_k (S positive values; None: off), daxm_set_step_weights."""
        if w is None:
            self._check(lib().daxm_set_step_weights(self._h, None))
            return
        w = np.ascontiguousarray(np.asarray(w, dtype=np.float64).reshape(-1))
        if w.shape[0] != self.n_steps:
            raise ValueError(f"{w.shape[0]} weights, the plan has {self.n_steps} steps")
        self._check(lib().daxm_set_step_weights(self._h, w.ctypes.data_as(C.POINTER(C.c_double))))

    def set_host_budget(self, device_bytes: int):
        """Cap the device memory reconstruct_host may hold (0 = no cap): above it the host path runs
        out of core through a two-slot ring of 128-aligned row bands (daxm_set_host_budget)."""
        if device_bytes < 0:
            raise ValueError("device_bytes must be >= 0")
        self._check(lib().daxm_set_host_budget(self._h, C.c_uint64(int(device_bytes))))

    def host_ring_info(self) -> dict:
        """Layout of the last reconstruct_host call (band_rows = n_bands = 0: it ran in core)."""
        v = [C.c_int64() for _ in range(3)]
        self._check(lib().daxm_host_ring_info(self._h, *[C.byref(x) for x in v]))
        return {"band_rows": v[0].value, "n_bands": v[1].value, "ring_bytes": v[2].value}

    def close(self):
        if self._h is not None and self._h.value:
            lib().daxm_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def create(g: dict, device: int = 0, rows: tuple | None = None) -> Plan:
    s, keep = make_geometry(g, rows)
    h = C.c_void_p()
    st = lib().daxm_create(C.byref(s), int(device), C.byref(h))
    del keep
    if st != 0:
        raise DaxmError(st, lib().daxm_create_error().decode())
    return Plan(h.value, device)


def reconstruct(plan: Plan, stack, out=None, stream=None):
    return plan.reconstruct(stack, out, stream)


def reconstruct_host(plan: Plan, stack, out=None, stream=None):
    return plan.reconstruct_host(stack, out, stream)
