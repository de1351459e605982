"""The C ABI without a GPU: the library loads, exports every symbol include/daxm.h
declares, the ctypes structs match the C layout, and argument validation that
needs no device returns the documented status codes."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "daxm.h")


@pytest.fixture(scope="module")
def daxm():
    from paper_2201_13309_b200 import _build
    _build.build_library()
    import paper_2201_13309_b200 as d
    return d


def declared_functions():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(daxm_\w+)\s*\(", txt, flags=re.M)))


def test_exports_every_declared_symbol(daxm):
    names = declared_functions()
    assert len(names) >= 10, names
    out = subprocess.check_output(["nm", "-D", "--defined-only", daxm.binding._LIB_PATH]).decode()
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = daxm.lib()
    for n in names:
        getattr(L, n)
    assert daxm.abi_version() == 1


def test_struct_layout_matches_header(daxm, tmp_path):
    src = tmp_path / "layout.c"
    fields_g = [f for f, _ in daxm.binding.Geometry._fields_]
    fields_s = [f for f, _ in daxm.binding.PlanStats._fields_]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "daxm.h"', "int main(void){"]
    lines.append('printf("%zu %zu\\n", sizeof(daxm_geometry), sizeof(daxm_plan_stats));')
    for f in fields_g:
        lines.append(f'printf("%zu\\n", offsetof(daxm_geometry, {f}));')
    for f in fields_s:
        lines.append(f'printf("%zu\\n", offsetof(daxm_plan_stats, {f}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).decode().split()]
    assert vals[0] == C.sizeof(daxm.binding.Geometry)
    assert vals[1] == C.sizeof(daxm.binding.PlanStats)
    offs = vals[2:]
    want = [getattr(daxm.binding.Geometry, f).offset for f in fields_g] + \
           [getattr(daxm.binding.PlanStats, f).offset for f in fields_s]
    assert offs == want


def _create_status(daxm, g, rows=None, device=0):
    try:
        daxm.create(g, device=device, rows=rows)
    except daxm.DaxmError as e:
        return e.status, e.detail
    return 0, ""


@pytest.mark.parametrize("mut,status", [
    (lambda g: g.update(wire_xyz=g["wire_xyz"][:1]), 1),                    # S < 2
    (lambda g: g.update(n_rows=0), 1),
    (lambda g: g.update(depth_res=0.0), 1),
    (lambda g: g.update(depth_res=-1.0), 1),
    (lambda g: g.update(depth_end=-60.0), 1),                               # end < start
    (lambda g: g.update(depth_res=0.3), 1),                                 # 100/0.3 not an integer
    (lambda g: g.update(wire_radius=0.0), 1),
    (lambda g: g.update(wire_radius=float("nan")), 1),
    (lambda g: g.update(beam_dir=(0.0, 0.0, 0.0)), 1),
    (lambda g: g.update(wire_axis=(0.0, 0.0, float("inf"))), 1),
    (lambda g: g.update(wire_axis=(0.0, 0.0, 1.0)), 1),                     # beam parallel to axis
    (lambda g: g.update(pitch_col=-5.0), 1),
    (lambda g: g.update(edge=7), 1),
    (lambda g: g.update(pixel_model=9), 1),
    (lambda g: g.update(wire_xyz=g["wire_xyz"][::-1][np.r_[0:5, 7, 6, 8:21]].copy()), 2),  # travel reverses
    (lambda g: g.update(wire_xyz=np.repeat(g["wire_xyz"][:1], 21, 0)), 2),  # no motion
])
def test_create_validation(daxm, mut, status):
    g = synth.geometry("C1")
    g["wire_xyz"] = g["wire_xyz"].copy()
    mut(g)
    st, detail = _create_status(daxm, g)
    assert st == status, (st, detail)
    assert detail


def test_band_and_null_validation(daxm):
    g = synth.geometry("C1")
    assert _create_status(daxm, g, rows=(10, 5))[0] == 1
    assert _create_status(daxm, g, rows=(0, 65))[0] == 1
    assert _create_status(daxm, g, rows=(-1, 5))[0] == 1
    L = daxm.lib()
    h = C.c_void_p()
    assert L.daxm_create(None, 0, C.byref(h)) == 1
    s, keep = daxm.binding.make_geometry(g)
    assert L.daxm_create(C.byref(s), 0, None) == 1
    assert L.daxm_plan_info(None, None, None, None) == 1
    assert L.daxm_reconstruct(None, None, 0, None, None) == 1
    L.daxm_destroy(None)
    assert L.daxm_status_string(3) == b"geometry error"


def test_along_axis_wire_offsets_are_allowed(daxm):
    """Wire centres may wander along the wire axis (depth does not depend on it): only the
    no-device status is returned, not a geometry error."""
    import torch
    g = synth.geometry("C1")
    W = g["wire_xyz"].copy()
    W[:, 0] += np.linspace(0, 40, W.shape[0])  # along a = x
    g["wire_xyz"] = W
    st, detail = _create_status(daxm, g)
    if torch.cuda.is_available():
        assert st == 0, detail
    else:
        assert st == 5 and "device" in detail
