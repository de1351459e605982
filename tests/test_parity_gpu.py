"""GPU vs fp64 oracle parity through the C ABI (BASELINE.json north_star tolerances).

* element by element on every config that the oracle finishes in seconds
  (C1, C2, C3 and ragged / banded / degenerate variants);
* at BASELINE.json's full sizes (C4, C5) in the launch configuration bench.py
  times, on sampled pixels the oracle computes one by one.
"""
import numpy as np
import pytest

import oracle
import parity
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def daxm():
    import torch
    from paper_2201_13309_b200 import _build
    _build.build_library()
    import paper_2201_13309_b200 as d
    assert torch.cuda.is_available()
    return d


def run_gpu(daxm, g, host_stack, rows=None):
    import torch
    with daxm.create(g, device=0, rows=rows) as plan:
        st = torch.from_numpy(np.ascontiguousarray(host_stack)).to("cuda:0")
        out = plan.reconstruct(st)
        torch.cuda.synchronize()
        stats = plan.stats()
        assert stats["lock_ring_violations"] == 0, stats  # counted by DAXM_*_CHECK builds only
        return out.cpu().numpy(), stats


@pytest.mark.parametrize("edge", ["leading", "trailing"])
@pytest.mark.parametrize("pixel_model", ["finite", "point"])
@pytest.mark.parametrize("dtype", ["f32", "u16"])
def test_c1_full(daxm, edge, pixel_model, dtype):
    g = synth.geometry("C1", edge=edge, pixel_model=pixel_model)
    maps = synth.make_maps("C1")
    host = synth.stack_numpy(maps, dtype, noise=True)
    gpu, st = run_gpu(daxm, g, host)
    ref = oracle.reconstruct(g, host)
    parity.check(gpu, ref, host, f"C1 {edge} {pixel_model} {dtype}")
    # the library's depth-model tolerance (MODEL_ERR_MAX = 2e-5 bins, daxm_internal.cuh)
    assert st["fit_model_err_bins"] < 2e-5 and st["fit_max_err_bins"] < 1e-4


@pytest.mark.parametrize("edge", ["leading", "trailing"])
def test_c2_full(daxm, edge):
    g = synth.geometry("C2", edge=edge)
    maps = synth.make_maps("C2")
    host = synth.stack_numpy(maps, "f32", noise=True)
    gpu, _ = run_gpu(daxm, g, host)
    ref = oracle.reconstruct(g, host)
    parity.check(gpu, ref, host, f"C2 {edge}")


def test_c2_peaks_only(daxm):
    """No noise: background pixels must come out exactly zero, peak pixels within tolerance."""
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "f32", noise=False)
    gpu, _ = run_gpu(daxm, g, host)
    ref = oracle.reconstruct(g, host)
    parity.check(gpu, ref, host, "C2 peaks")
    flat = parity.abs_dI(host) == 0
    assert (gpu[:, flat] == 0).all()
    assert np.abs(gpu).max() > 100


def test_c3_full_u16(daxm):
    g = synth.geometry("C3")
    maps = synth.make_maps("C3")
    host = synth.stack_numpy(maps, "u16", noise=False)
    gpu, _ = run_gpu(daxm, g, host)
    ref = oracle.reconstruct(g, host)
    parity.check(gpu, ref, host, "C3")


def _sample_pixels(cfg, maps, n_rand, rng):
    n = cfg.n
    js = list(rng.integers(0, n, n_rand))
    is_ = list(rng.integers(0, n, n_rand))
    peak = np.argwhere(maps.amp > 0)
    if len(peak):
        sel = peak[rng.choice(len(peak), size=min(600, len(peak)), replace=False)]
        js += list(sel[:, 0])
        is_ += list(sel[:, 1])
    for (j, i) in [(0, 0), (0, n - 1), (n - 1, 0), (n - 1, n - 1), (31, 32), (32, 31), (n // 2, n // 2)]:
        js.append(j)
        is_.append(i)
    return np.array(js), np.array(is_)


@pytest.mark.parametrize("name,noise,dtype,fraction", [
    ("C3", True, None, None), ("C4", True, None, None), ("C5", False, None, None), ("C5", True, None, None),
    # fp32 stacks at full size (C5 is quoted for u16 and fp32)
    ("C4", True, "f32", None), ("C5", True, "f32", None),
    # intensity cutoff at full size, as bench.py --fraction runs it (reading R14)
    ("C5", False, None, 0.05), ("C5", True, None, 0.25), ("C4", True, None, 0.5)])
def test_full_size_sampled(daxm, name, noise, dtype, fraction):
    """BASELINE.json full sizes, stack generated on the GPU exactly as bench.py does;
    sampled pixels recomputed by the oracle from the generator's per-pixel series.
    With a pixel fraction the cutoff is daxm_select_cutoff's (checked against the oracle's
    order statistic of the same first image) and the oracle zeroes the inactive pixels."""
    import dataclasses

    import torch
    cfg = synth.get_config(name)
    if dtype:
        cfg = dataclasses.replace(cfg, dtype=dtype)
    g = synth.geometry(cfg)
    maps = synth.make_maps(cfg)
    rng = np.random.default_rng(7 + cfg.number)
    js, is_ = _sample_pixels(cfg, maps, 1500, rng)
    cut = None
    with daxm.create(g, device=0) as plan:
        stack = synth.stack_torch(maps, cfg.dtype, "cuda:0", noise=noise)
        if fraction is not None:
            cut = plan.select_cutoff(stack, fraction)
            first = stack[0].cpu().numpy()
            assert np.float32(cut) == np.float32(oracle.select_cutoff(first, fraction))
            plan.set_cutoff(cut)
            # the sample must hold both active and inactive pixels
            act = oracle.active_pixels(first[js, is_], cut)
            assert act.any() and (~act).any()
        out = plan.reconstruct(stack)
        torch.cuda.synchronize()
        if name == "C4":  # the production row kernel, not a fallback
            assert plan.stats()["row_path"] == 1
        jt = torch.from_numpy(js).cuda()
        it = torch.from_numpy(is_).cuda()
        gpu = out[:, jt, it].cpu().numpy()  # [M, n]
        del stack, out
        torch.cuda.empty_cache()
    series = synth.pixel_series(maps, js, is_, cfg.dtype, noise=noise)  # [n, S]
    ref = oracle.reconstruct_pixels(g, js, is_, series).T
    if cut is not None:
        ref[:, ~oracle.active_pixels(series[:, 0], cut)] = 0.0
    parity.check(gpu, ref, series.T, f"{name} {cfg.dtype} sampled fraction={fraction}")


@pytest.mark.parametrize("col0,expect", [(1344, "wide"), (1856, "overlap"), (1700, "mixed"), (256, "separated")])
@pytest.mark.parametrize("dtype", ["u16", "f32"])
def test_c5_regions_element_by_element(daxm, col0, expect, dtype):
    """64 x 128 windows of the C5 detector (synth.crop_geometry: the same pixel positions, so the
    same depth spans and step spacings) where the edge spans are 2-3 bins wide ("wide"), where
    consecutive spans overlap ("overlap", up to 1.5x the step), across the transition ("mixed")
    and in the separated regime: every row tile runs the row kernel -- the general-span variant
    in the first three -- and every output element is within tolerance of the
    oracle's."""
    g = synth.crop_geometry("C5", 1000, col0, 64, 128)
    S = g["wire_xyz"].shape[0]
    rng = np.random.default_rng(col0)
    host = (20000 + rng.integers(-3000, 3000, (S, 64, 128))).astype(np.uint16 if dtype == "u16" else np.float32)
    gpu, st = run_gpu(daxm, g, host)
    assert st["row_path"] == 1, st
    if expect == "separated":
        assert st["row_tiles_gen"] == 0
    else:
        assert st["row_tiles_gen"] > 0, st
    parity.check(gpu, oracle.reconstruct(g, host), host, f"C5 window col0={col0} {dtype}")


@pytest.mark.parametrize("name,dtype", [("C3", "u16"), ("C2", "f32")])
def test_zero_skip_equals_full_run(daxm, name, dtype, monkeypatch):
    """The row kernel's exact zero-dI skip (tiles whose intensities never change write zeros
    without running the deposit) gives the same values as running every tile in full, and the
    oracle's exact zeros on the constant pixels (noise-free stacks: most tiles constant)."""
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=False)
    skip, st = run_gpu(daxm, g, host)
    assert st["row_path"] == 1
    monkeypatch.setenv("DAXM_NO_ZERO_SKIP", "1")
    full, _ = run_gpu(daxm, g, host)
    assert np.array_equal(skip, full)
    flat = parity.abs_dI(host) == 0
    assert flat.mean() > 0.5 and (skip[:, flat] == 0).all()
    parity.check(skip, oracle.reconstruct(g, host), host, f"{name} zero skip")


@pytest.mark.parametrize("name,dtype,pixel_model", [("C1", "f32", "finite"), ("C1", "u16", "point"),
                                                    ("C2", "f32", "finite"), ("C3", "u16", "finite")])
def test_both_edges_mode(daxm, name, dtype, pixel_model):
    """edge = "both" (reading R16): the leading child plan stores the reconstruction of the
    intensity decreases, the trailing child adds (TMA reduce-add) that of the increases; element
    by element against the oracle's both-edges mode, whose pins are tests/test_oracle_both.py."""
    g = synth.geometry(name, edge="both", pixel_model=pixel_model)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    gpu, st = run_gpu(daxm, g, host)
    assert st["row_path"] == 1, st
    ref = oracle.reconstruct(g, host)
    parity.check(gpu, ref, host, f"{name} both edges")
    # the mode is really both: not the leading reconstruction
    lead = oracle.reconstruct(synth.geometry(name, pixel_model=pixel_model), host)
    assert np.abs(ref - lead).max() > 10 * np.abs(gpu - ref).max()


def test_both_edges_host_path_and_cutoff(daxm):
    """The both-edges mode through daxm_reconstruct_host (band pipeline) and with a cutoff."""
    import torch
    g = synth.geometry("C3", edge="both")
    host = synth.stack_numpy(synth.make_maps("C3"), "u16", noise=True)
    ref = oracle.reconstruct(g, host)
    cut = oracle.select_cutoff(host[0], 0.3)
    with daxm.create(g, device=0) as plan:
        out = np.asarray(plan.reconstruct_host(host))
        parity.check(out, ref, host, "C3 both host")
        plan.set_cutoff(cut)
        dev = plan.reconstruct(torch.from_numpy(host).cuda()).cpu().numpy()
    ref[:, ~oracle.active_pixels(host[0], cut)] = 0
    parity.check(dev, ref, host, "C3 both cutoff")


# ------------------------------------------------------------------ edge cases

def test_ragged_detector(daxm):
    """Sizes that are not multiples of the 32x32 tile (partial tiles on both axes)."""
    g = synth.geometry("C2", n_rows=77, n_cols=45)
    g["wire_xyz"] = synth.wire_positions(61, t_range=(40.0, 1040.0))
    rng = np.random.default_rng(3)
    host = (1000 + rng.integers(-300, 300, (61, 77, 45))).astype(np.float32)
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, "ragged")


@pytest.mark.parametrize("name,edge", [("C1", "leading"), ("C2", "leading"), ("C2", "trailing"), ("C3", "leading"),
                                       ("C4", "leading")])
def test_row_path_admits_every_tile(daxm, name, edge):
    """The production row-segment kernel (deposit_row.cu) takes every row tile of the C1-C4
    workloads (so the parity tests of those configs exercise it, not the fallback kernels)."""
    import os
    if os.environ.get("DAXM_NO_ROW"):
        pytest.skip("row path disabled by DAXM_NO_ROW")
    with daxm.create(synth.geometry(name, edge=edge), device=0) as plan:
        st = plan.stats()
    assert st["row_path"] == 1 and st["row_tiles_general"] == 0, {k: st[k] for k in st if k.startswith("row_")}


def test_row_bands(daxm):
    """Row bands (the multi-GPU sharding).  Bands aligned to the 128-row tile reproduce the
    full-detector plan bit for bit (every tile reference is global); bands starting inside a
    tile run that tile through the general kernel and must still match the oracle."""
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "f32", noise=True)
    full, _ = run_gpu(daxm, g, host)
    for (r0, r1) in [(0, 256), (256, 512), (128, 384), (384, 500)]:
        band, _ = run_gpu(daxm, g, host[:, r0:r1], rows=(r0, r1))
        assert np.array_equal(band, full[:, r0:r1]), (r0, r1)
    ref = oracle.reconstruct(g, host)
    for (r0, r1) in [(100, 300), (511, 512), (5, 37)]:
        band, st = run_gpu(daxm, g, host[:, r0:r1], rows=(r0, r1))
        assert st["general_tiles_f32"] > 0
        parity.check(band, ref[:, r0:r1], host[:, r0:r1], f"band {r0}-{r1}")


def test_no_pixel_reaches_the_bins(daxm):
    g = synth.geometry("C1")
    g["depth_start"], g["depth_end"] = 5000.0, 5100.0
    host = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
    gpu, st = run_gpu(daxm, g, host)
    assert not gpu.any() and st["contrib_pairs"] == 0


def test_single_bin_and_two_steps(daxm):
    g = synth.geometry("C1")
    g["depth_start"] = g["depth_end"] = 3.0
    g["depth_res"] = 40.0
    host = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, "M=1")
    g2 = synth.geometry("C1")
    g2["wire_xyz"] = g2["wire_xyz"][[8, 12]].copy()
    h2 = host[[8, 12]].copy()
    gpu2, _ = run_gpu(daxm, g2, h2)
    parity.check(gpu2, oracle.reconstruct(g2, h2), h2, "S=2")


@pytest.mark.parametrize("name,dtype,edge", [("C1", "f32", "leading"), ("C2", "u16", "trailing"),
                                             ("C2", "f32", "both")])
def test_step_weights(daxm, name, dtype, edge):
    """Per-step intensity normalisation (reading R17, daxm_set_step_weights): element by element
    against the oracle with the same weights; tolerance denominators from the normalised images.
    Switching the weights off returns the fast path's result."""
    import torch
    g = synth.geometry(name, edge=edge)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    S = host.shape[0]
    w = np.random.default_rng(17).uniform(0.85, 1.2, S)
    with daxm.create(g, device=0) as plan:
        st = torch.from_numpy(host).cuda()
        plain = plan.reconstruct(st).cpu().numpy()
        plan.set_step_weights(w)
        gpu = plan.reconstruct(st).cpu().numpy()
        plan.set_step_weights(None)
        again = plan.reconstruct(st).cpu().numpy()
        assert np.array_equal(again, plain)
        with pytest.raises(daxm.DaxmError):
            plan.set_step_weights(np.full(S, -1.0))
    ref = oracle.reconstruct(dict(g, step_weight=w), host)
    parity.check(gpu, ref, host.astype(np.float64) * w[:, None, None], f"{name} {edge} step weights")
    assert np.abs(gpu - plain).max() > 1.0


@pytest.mark.parametrize("pixel_model", ["finite", "point"])
def test_repeated_wire_positions(daxm, pixel_model):
    """Zero-travel pairs: POINT mode gives the degenerate delta (z1 == z4, reading R8)."""
    g = synth.geometry("C1", pixel_model=pixel_model)
    W = g["wire_xyz"]
    g["wire_xyz"] = W[[0, 1, 2, 3, 4, 5, 6, 7, 8, 8, 9, 10, 10, 11, 12, 13, 14, 15, 16, 17, 18]].copy()
    host = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, f"repeated {pixel_model}")


def test_reversed_scan_direction(daxm):
    """Wire moving the other way (depth decreasing with the step index)."""
    g = synth.geometry("C2", edge="leading")
    g["wire_xyz"] = g["wire_xyz"][::-1].copy()
    host = synth.stack_numpy(synth.make_maps("C2"), "f32", noise=True)[::-1].copy()
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, "reversed")


def test_u16_extremes(daxm):
    g = synth.geometry("C1")
    rng = np.random.default_rng(5)
    host = rng.choice(np.array([0, 65535, 1, 65534], dtype=np.uint16), size=(21, 64, 64))
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, "u16 extremes")


def test_host_path_matches_device_path(daxm):
    import torch
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True)
    with daxm.create(g, device=0) as plan:
        dev = plan.reconstruct(torch.from_numpy(host).cuda())
        torch.cuda.synchronize()
        hp = plan.reconstruct_host(torch.from_numpy(host).pin_memory())
        assert torch.equal(dev.cpu(), hp)


def test_bad_pointers_on_device(daxm):
    import torch
    g = synth.geometry("C1")
    with daxm.create(g, device=0) as plan:
        st = torch.zeros((21, 64, 64), dtype=torch.float32, device="cuda")
        with pytest.raises(ValueError):
            plan.reconstruct(st.to(torch.float64))
        with pytest.raises(ValueError):
            plan.reconstruct(st, out=torch.empty((3, 3), device="cuda"))
        with pytest.raises(daxm.DaxmError):
            daxm.lib()  # library present
            import ctypes as C
            st_code = daxm.lib().daxm_reconstruct(plan._h, C.c_void_p(st.data_ptr() + 4), 1,
                                                  C.c_void_p(st.data_ptr()), None)
            plan._check(st_code)


@pytest.mark.parametrize("name,dtype", [("C1", "f32"), ("C2", "f32"), ("C2", "u16")])
def test_general_kernel_parity(daxm, name, dtype, monkeypatch):
    """The general (any-geometry) deposit kernel on its own: DAXM_FORCE_GENERAL routes every tile to it."""
    monkeypatch.setenv("DAXM_FORCE_GENERAL", "1")
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, f"{name} general")


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_benchmark_configs_take_the_fast_path(daxm, name):
    """Every tile of these BASELINE configs is 'separated' and fits the input ring, so bench.py times
    the TMA-pipelined kernel alone.  (C5's finest bins make the pixel-edge span exceed the
    per-step sweep on the detector's shallow side: those tiles run the general kernel, see
    test_c5_general_tiles_are_the_overlapping_ones.)"""
    cfg = synth.get_config(name)
    with daxm.create(synth.geometry(cfg), device=0) as plan:
        st = plan.stats()
    key = "general_tiles_u16" if cfg.dtype == "u16" else "general_tiles_f32"
    assert st[key] == 0, {k: st[k] for k in ("nonseparated_tiles", "ring_need_max", key)}


def test_c5_overlapping_tiles_use_the_ramp_superposition_kernel(daxm):
    """C5's finest bins make the pixel-edge span exceed the per-step sweep on the detector's
    shallow side: those tiles run the step-locked ramp-superposition kernel (deposit_lock, OV);
    only tiles mixing both regimes fall back to the general kernel."""
    cfg = synth.get_config("C5")
    with daxm.create(synth.geometry(cfg), device=0) as plan:
        st = plan.stats()
    assert st["overlap_tiles"] > 0
    assert st["lock_tiles_overlap"] == st["overlap_tiles"], st
    assert st["general_tiles_u16"] == st["nonseparated_tiles"] - st["overlap_tiles"]
    assert st["general_tiles_u16"] < st["n_tiles"] // 20


@pytest.mark.parametrize("dtype", ["u16", "f32"])
def test_overlap_regime_dual_walk_fallback(daxm, dtype, monkeypatch):
    """DAXM_NO_LOCK_OV keeps the overlapping tiles on the fast kernel's dual ramp walk: both
    algebras of the overlap regime match the oracle."""
    monkeypatch.setenv("DAXM_NO_LOCK_OV", "1")
    g = synth.geometry("C2", n_rows=96, n_cols=64)
    g["wire_xyz"] = synth.wire_positions(1601, t_range=(40.0, 1040.0))
    g["depth_res"] = 0.5
    rng = np.random.default_rng(18)
    host = (3000 + rng.integers(-400, 400, (1601, 96, 64))).astype(np.uint16 if dtype == "u16" else np.float32)
    gpu, st = run_gpu(daxm, g, host)
    assert st["overlap_tiles"] == st["n_tiles"] and st["lock_tiles_overlap"] == 0, st
    parity.check(gpu, oracle.reconstruct(g, host), host, f"overlap dual walk {dtype}")


@pytest.mark.parametrize("dtype", ["u16", "f32"])
def test_overlap_regime_parity(daxm, dtype):
    """Many fine wire steps on a coarse-pitch detector: every pixel's edge span (0.68 um) exceeds
    the per-step sweep (0.24-0.6 um) -> all tiles overlapping, all in deposit_lock (OV)."""
    g = synth.geometry("C2", n_rows=96, n_cols=64)
    g["wire_xyz"] = synth.wire_positions(1601, t_range=(40.0, 1040.0))
    g["depth_res"] = 0.5
    rng = np.random.default_rng(17)
    host = (3000 + rng.integers(-400, 400, (1601, 96, 64))).astype(np.uint16 if dtype == "u16" else np.float32)
    gpu, st = run_gpu(daxm, g, host)
    assert st["overlap_tiles"] == st["n_tiles"], st
    assert st["lock_tiles_overlap"] == st["n_tiles"], st  # the ramp-superposition kernel
    parity.check(gpu, oracle.reconstruct(g, host), host, f"overlap {dtype}")


def test_host_path_pipelined_bands(daxm):
    """daxm_reconstruct_host pipelines row bands over three streams; a band plan that starts
    inside a tile must still reproduce its device-path output exactly."""
    import torch
    g = synth.geometry("C3")
    host = synth.stack_numpy(synth.make_maps("C3"), "u16", noise=True)
    for rows in [(0, 1024), (70, 901), (71, 899)]:  # (an odd start: row tiles start at row 71)
        band = np.ascontiguousarray(host[:, rows[0]:rows[1]])
        with daxm.create(g, device=0, rows=rows) as plan:
            dev = plan.reconstruct(torch.from_numpy(band).cuda())
            torch.cuda.synchronize()
            hp = plan.reconstruct_host(torch.from_numpy(band).pin_memory())
            hp2 = plan.reconstruct_host(band)  # pageable host memory works too
            assert torch.equal(dev.cpu(), hp) and torch.equal(hp, hp2)


def test_host_path_out_of_core(daxm):
    """Out-of-core host path (the paper's row chunking P:L182-215): under a
    device budget smaller than stack + output the call streams 128-row bands through a two-slot
    ring (device memory O(band)) and returns the whole-plan device-path output bit for bit --
    also for a plan that starts inside a band, under a cutoff, and in both-edges mode; a budget
    that cannot hold two 128-row slots is OUT_OF_MEMORY."""
    import torch
    g = synth.geometry("C3")
    host = synth.stack_numpy(synth.make_maps("C3"), "u16", noise=True)
    in_b, out_b = host.nbytes, 201 * 1024 * 1024 * 4
    for rows in [(0, 1024), (70, 901)]:
        band = np.ascontiguousarray(host[:, rows[0]:rows[1]])
        with daxm.create(g, device=0, rows=rows) as plan:
            dev = plan.reconstruct(torch.from_numpy(band).cuda()).cpu()
            budget = (in_b + out_b) // 3  # the whole stack + output does not fit
            plan.set_host_budget(budget)
            hp = plan.reconstruct_host(torch.from_numpy(band).pin_memory())
            info = plan.host_ring_info()
            assert info["band_rows"] >= 128 and info["band_rows"] % 128 == 0, info
            assert info["n_bands"] >= 2 and 0 < info["ring_bytes"] <= budget, info
            assert torch.equal(dev, hp), rows
            # cutoff through the ring = cutoff on the device path
            c = float(np.quantile(band[0], 0.7))
            plan.set_cutoff(c)
            hc = plan.reconstruct_host(band)
            dc = plan.reconstruct(torch.from_numpy(band).cuda()).cpu()
            assert torch.equal(dc, hc) and not torch.equal(hc, hp)
            plan.set_cutoff(None)
            plan.set_host_budget(0)  # back in core
            assert torch.equal(plan.reconstruct_host(band), dev) and plan.host_ring_info()["n_bands"] == 0
            plan.set_host_budget(1 << 20)
            with pytest.raises(daxm.DaxmError, match="OUT_OF_MEMORY|budget"):
                plan.reconstruct_host(band)
    gb = synth.geometry("C2", edge="both")
    hb = synth.stack_numpy(synth.make_maps("C2"), "f32", noise=True)
    with daxm.create(gb, device=0) as plan:
        dev = plan.reconstruct(torch.from_numpy(hb).cuda()).cpu()
        plan.set_host_budget((hb.nbytes + dev.numel() * 4) // 2)
        hp = plan.reconstruct_host(hb)
        assert plan.host_ring_info()["n_bands"] >= 2 and torch.equal(dev, hp)


@pytest.mark.parametrize("name,dtype", [("C2", "f32"), ("C3", "u16")])
def test_depth_profile(daxm, name, dtype):
    """daxm_depth_profile = the paper's image_set.depth_intensity: per-bin totals of the
    reconstruction, checked against the oracle's totals."""
    import torch
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    with daxm.create(g, device=0) as plan:
        out = plan.reconstruct(torch.from_numpy(host).cuda())
        prof = plan.depth_profile(out).cpu().numpy()
        again = out.double().sum(dim=(1, 2)).cpu().numpy()
    ref = oracle.reconstruct(g, host).sum(axis=(1, 2))
    scale = parity.abs_dI(host).sum()
    assert np.allclose(prof, again, rtol=1e-9, atol=1e-6 * scale)
    assert np.abs(prof - ref).max() <= 1e-5 * scale


@pytest.mark.parametrize("name,dtype,fraction", [("C1", "f32", None), ("C2", "f32", None), ("C3", "u16", None),
                                                 ("C3", "u16", 0.2), ("C2", "u16", "noise-free")])
def test_fused_profile(daxm, name, dtype, fraction, monkeypatch):
    """daxm_reconstruct_profile: the row kernel's fused per-tile plane sums + tile reduction give
    the oracle's depth profile (oracle.depth_profile, pinned by conservation), the same output as
    daxm_reconstruct, and the unfused profile of that output; also with a cutoff and with the
    zero-dI skip's dead tiles (noise-free stack)."""
    import torch
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=fraction != "noise-free")
    ref_out = oracle.reconstruct(g, host)
    with daxm.create(g, device=0) as plan:
        assert plan.stats()["row_path"] == 1
        st = torch.from_numpy(host).cuda()
        if isinstance(fraction, float):
            cut = oracle.select_cutoff(host[0], fraction)
            plan.set_cutoff(cut)
            ref_out[:, ~oracle.active_pixels(host[0], cut)] = 0
        out, prof = plan.reconstruct_profile(st)
        plain = plan.reconstruct(st)
        unfused = plan.depth_profile(plain)
        assert torch.equal(out, plain)
        prof, unfused = prof.cpu().numpy(), unfused.cpu().numpy()
    scale = parity.abs_dI(host).sum()
    ref = oracle.depth_profile(ref_out)
    assert np.abs(prof - ref).max() <= 1e-5 * scale
    assert np.allclose(prof, unfused, rtol=1e-6, atol=1e-7 * scale)
    parity.check(out.cpu().numpy(), ref_out, host, f"{name} fused profile output")


@pytest.mark.parametrize("name,dtype", [("C2", "f32"), ("C3", "u16")])
@pytest.mark.parametrize("fraction", [0.003, 0.25, 1.0])
def test_select_cutoff_matches_oracle(daxm, name, dtype, fraction):
    """Pixel percentage (reading R14): the device radix select returns exactly the
    oracle's k-th largest first-step intensity."""
    import torch
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    if dtype == "f32":
        host[0, 5, 7] = np.nan
        host[0, 9, 9] = -np.inf
    with daxm.create(g, device=0) as plan:
        c = plan.select_cutoff(torch.from_numpy(host).cuda(), fraction)
    assert c == oracle.select_cutoff(host[0], fraction)


@pytest.mark.parametrize("name,dtype,fraction", [("C3", "u16", 0.25), ("C2", "f32", 0.003), ("C2", "f32", 1.0)])
def test_select_cutoff_sharded(daxm, name, dtype, fraction):
    """daxm_select_cutoff_sharded with two row-band plans in lock step (two threads; the
    reduce callback sums their digit histograms at a barrier) = the oracle's order statistic
    of the whole first image, on both shards."""
    import threading

    import torch
    g = synth.geometry(name)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    R = g["n_rows"]
    bands = [(0, R // 2), (R // 2, R)]
    barrier = threading.Barrier(2, timeout=120)
    slots = [None, None]
    res = [None, None]

    def worker(i):
        b0, b1 = bands[i]
        with daxm.create(g, device=0, rows=(b0, b1)) as plan:
            st = torch.from_numpy(np.ascontiguousarray(host[:, b0:b1])).to("cuda:0")
            stream = torch.cuda.Stream(device=0)

            def reduce(h):
                slots[i] = h.copy()
                barrier.wait()
                tot = slots[0] + slots[1]
                barrier.wait()
                h[:] = tot
            with torch.cuda.stream(stream):
                res[i] = plan.select_cutoff_sharded(st, fraction, R * g["n_cols"], reduce, stream)
    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    ref = oracle.select_cutoff(host[0], fraction)
    assert res[0] == res[1] and np.float32(res[0]) == np.float32(ref), (res, ref)


@pytest.mark.parametrize("case", ["C2-f32", "C3-u16", "C3-u16-band", "C2-u16-general", "overlap-u16", "C3-u16-host"])
def test_cutoff_parity(daxm, case, monkeypatch):
    """Intensity cutoff (d_cutoff; reading R14): pixels below it are not processed and
    read as 0, all others are bit-for-bit what the unrestricted run gives (same kernels); tiles
    with no active pixel skip their input stream entirely."""
    import torch
    name, dtype = case.split("-")[:2]
    rows = None
    if name == "overlap":
        g = synth.geometry("C2", n_rows=96, n_cols=64)
        g["wire_xyz"] = synth.wire_positions(1601, t_range=(40.0, 1040.0))
        g["depth_res"] = 0.5
        rng = np.random.default_rng(18)
        host = (3000 + rng.integers(-400, 400, (1601, 96, 64))).astype(np.uint16)
    else:
        g = synth.geometry(name)
        host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    if case.endswith("general"):
        monkeypatch.setenv("DAXM_FORCE_GENERAL", "1")
    if case.endswith("band"):
        rows = (128, 901)
    band = np.ascontiguousarray(host[:, rows[0]:rows[1]] if rows else host)
    with daxm.create(g, device=0, rows=rows) as plan:
        dev = torch.from_numpy(band).cuda()
        full = plan.reconstruct(dev).cpu().numpy()
        c = plan.select_cutoff(dev, 0.1)
        plan.set_cutoff(c)
        part = (plan.reconstruct_host(band) if case.endswith("host") else plan.reconstruct(dev).cpu()).numpy()
        plan.set_cutoff(None)
        again = plan.reconstruct(dev).cpu().numpy()
    act = oracle.active_pixels(band[0], c)
    assert 0.1 * act.size <= act.sum() < 0.5 * act.size
    assert np.array_equal(part[:, act], full[:, act])
    assert not part[:, ~act].any()
    assert np.array_equal(again, full)
    if name in ("C2", "overlap"):  # small enough for the whole oracle
        ref = oracle.reconstruct_cutoff(g, host, c, rows=rows)
        if rows:
            ref = ref[:, rows[0]:rows[1]]
        parity.check(part, ref, band, f"cutoff {case}")


def test_cutoff_skips_inactive_tiles(daxm):
    """A cutoff above every pixel but a few leaves almost every tile without work: the output is
    exactly zero there and the few active pixels still match the unrestricted run."""
    import torch
    g = synth.geometry("C3")
    host = synth.stack_numpy(synth.make_maps("C3"), "u16", noise=True)
    host[0, 300:303, 500:502] = 65535
    with daxm.create(g, device=0) as plan:
        dev = torch.from_numpy(host).cuda()
        full = plan.reconstruct(dev)
        plan.set_cutoff(65535)
        part = plan.reconstruct(dev)
        torch.cuda.synchronize()
    act = host[0] == 65535
    assert act.sum() == 6
    assert torch.equal(part[:, torch.from_numpy(act).cuda()], full[:, torch.from_numpy(act).cuda()])
    assert int(torch.count_nonzero(part[:, torch.from_numpy(~act).cuda()])) == 0


@pytest.mark.parametrize("rows,host_path", [(None, False), ((100, 1000), False), ((100, 1000), True)])
def test_cutoff_dead_tiles_written(daxm, rows, host_path):
    """Tiles with no pixel above the cutoff are skipped by every deposit kernel and their planes
    are written as zeros by the row-wise zero fill: an output buffer pre-filled with NaN must come
    back exactly zero there (band starting inside a tile, device and host paths), and live tiles
    bit for bit as the unrestricted run."""
    import torch
    g = synth.geometry("C3")
    host = synth.stack_numpy(synth.make_maps("C3"), "u16", noise=True)
    host[0] = 100
    host[0, 130:140, 17:19] = 5000    # live tiles in the first (partial) tile row of the band
    host[0, 600:900:37, 400:1000:53] = 5000  # scattered live pixels
    band = np.ascontiguousarray(host[:, rows[0]:rows[1]] if rows else host)
    with daxm.create(g, device=0, rows=rows) as plan:
        dev = torch.from_numpy(band).cuda()
        full = plan.reconstruct(dev).cpu()
        plan.set_cutoff(5000)
        if host_path:
            out = torch.full(plan.output_shape(), float("nan"), dtype=torch.float32).pin_memory()
            plan.reconstruct_host(torch.from_numpy(band).pin_memory(), out=out)
            part = out
        else:
            out = torch.full(plan.output_shape(), float("nan"), dtype=torch.float32, device="cuda")
            plan.reconstruct(dev, out=out)
            part = out.cpu()
        torch.cuda.synchronize()
    act = torch.from_numpy(band[0] == 5000)
    assert int(act.sum()) > 0
    assert torch.equal(part[:, act], full[:, act])
    assert not torch.isnan(part).any()
    assert int(torch.count_nonzero(part[:, ~act])) == 0


@pytest.mark.parametrize("name,dtype,edge", [("C1", "f32", "leading"), ("C2", "u16", "leading"),
                                             ("C2", "f32", "trailing")])
def test_general_wire_path(daxm, name, dtype, edge):
    """a jittered (non-straight) scan has no travel polynomial; the plan builds the
    exact per-step depth table and the general kernel reproduces the oracle (which uses the
    actual W_k)."""
    cfg = synth.get_config(name)
    g = synth.geometry(name, edge=edge)
    g["wire_xyz"] = synth.jittered_wire_positions(cfg.n_steps, t_range=cfg.t_range, amp_um=0.3)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    gpu, st = run_gpu(daxm, g, host)
    assert st["depth_table_bytes"] > 0 and st[f"general_tiles_{dtype}"] == st["n_tiles"], st
    parity.check(gpu, oracle.reconstruct(g, host), host, f"{name} jittered {edge}")


def test_forced_table_equals_model_path(daxm, monkeypatch):
    """The exact-table path on a straight scan (DAXM_FORCE_TABLE) against the oracle and against
    the polynomial-model fast path."""
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True)
    fast, st0 = run_gpu(daxm, g, host)
    monkeypatch.setenv("DAXM_FORCE_TABLE", "1")
    tab, st1 = run_gpu(daxm, g, host)
    assert st0["depth_table_bytes"] == 0 and st1["depth_table_bytes"] > 0
    parity.check(tab, oracle.reconstruct(g, host), host, "C2 forced table")
    d = parity.abs_dI(host)
    assert (np.abs(tab - fast) <= 2e-4 * d[None]).all()


def test_general_wire_path_full_size_sampled(daxm):
    """C3-size jittered scan through the table path; sampled pixels against the oracle."""
    import torch
    cfg = synth.get_config("C3")
    g = synth.geometry("C3")
    g["wire_xyz"] = synth.jittered_wire_positions(cfg.n_steps, t_range=cfg.t_range, amp_um=0.2, seed=7)
    maps = synth.make_maps("C3")
    rng = np.random.default_rng(5)
    js, is_ = _sample_pixels(cfg, maps, 300, rng)
    with daxm.create(g, device=0) as plan:
        assert plan.stats()["depth_table_bytes"] > 0
        out = plan.reconstruct(synth.stack_torch(maps, "u16", "cuda:0", noise=True))
        gpu = out[:, torch.from_numpy(js).cuda(), torch.from_numpy(is_).cuda()].cpu().numpy()  # [M, n]
    ser = synth.pixel_series(maps, js, is_, "u16", noise=True)
    ref = oracle.reconstruct_pixels(g, js, is_, ser).T
    parity.check(gpu, ref, ser.T, "C3 jittered sampled")


# ------------------------------------------------------------------ step-locked kernel

@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_lock_kernel_owns_separated_tiles(daxm, name):
    """The pre-pass admits (nearly) every separated tile of the benchmark configs to the
    step-locked kernel, and its ring-capacity counter stays 0 after a reconstruction."""
    import torch
    cfg = synth.get_config(name)
    g = synth.geometry(cfg)
    with daxm.create(g, device=0) as plan:
        st = plan.stats()
        n_lock = st["lock_tiles_small"] + st["lock_tiles_large"]
        n_sep = st["n_tiles"] - st["nonseparated_tiles"]
        assert n_lock >= 0.9 * n_sep, st
        if name in ("C2", "C3"):
            stack = torch.from_numpy(synth.stack_numpy(synth.make_maps(cfg), cfg.dtype, noise=True)).cuda()
        else:
            stack = synth.stack_torch(synth.make_maps(cfg), cfg.dtype, "cuda:0", noise=True)
        plan.reconstruct(stack)
        torch.cuda.synchronize()
        assert plan.stats()["lock_ring_violations"] == 0


@pytest.mark.parametrize("case", ["C1-f32", "C1-u16-point", "C2-f32-trailing", "C3-u16"])
def test_fast_kernel_without_lock(daxm, case, monkeypatch):
    """DAXM_NO_LOCK routes the separated tiles back to the bin-major fast kernel: both
    schedules of the same deposit algebra match the oracle."""
    monkeypatch.setenv("DAXM_NO_LOCK", "1")
    parts = case.split("-")
    name, dtype = parts[0], parts[1]
    edge = "trailing" if "trailing" in parts else "leading"
    pm = "point" if "point" in parts else "finite"
    g = synth.geometry(name, edge=edge, pixel_model=pm)
    host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
    gpu, _ = run_gpu(daxm, g, host)
    parity.check(gpu, oracle.reconstruct(g, host), host, f"{case} fast (no lock)")


def test_lock_kernel_sparse_and_cutoff(daxm):
    """Sparse stack (most pixels have dI = 0 everywhere) with an intensity cutoff: inactive
    walks and zero planes through the step-locked kernel."""
    import torch
    g = synth.geometry("C3")
    maps = synth.make_maps("C3")
    host = synth.stack_numpy(maps, "u16", noise=False)
    with daxm.create(g, device=0) as plan:
        st = torch.from_numpy(host).cuda()
        cut = plan.select_cutoff(st, 0.05)
        plan.set_cutoff(cut)
        out = plan.reconstruct(st)
        torch.cuda.synchronize()
        gpu = out.cpu().numpy()
        assert plan.stats()["lock_ring_violations"] == 0
    ref = oracle.reconstruct_cutoff(g, host, cut)
    parity.check(gpu, ref, host, "C3 sparse cutoff (lock)")


def test_lock_ring_check_build(tmp_path):
    """A DAXM_LOCK_CHECK=1 build of the library counts every write past the recycled part of
    a warp's output ring; the pre-pass admission must make that count 0 on every config."""
    import json
    import os
    import subprocess
    import sys
    from paper_2201_13309_b200 import _build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = _build.build_library(out=str(tmp_path / "libdaxm_lockcheck.so"), defines=["DAXM_LOCK_CHECK=1"])
    env = dict(os.environ, DAXM_LIBRARY=lib)
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "lock_check.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res and all(v["lock_ring_violations"] == 0 for v in res.values()), res
    assert all(v["lock_tiles_small"] + v["lock_tiles_large"] > 0 for v in res.values()), res


def test_reconstruct_is_graph_capturable(daxm):
    """daxm_reconstruct is stream-ordered and allocation-free: captured into a CUDA graph (C5:
    three tile classes whose launches fork onto the plan's streams and join back) and replayed,
    it reproduces the eager result bit for bit."""
    import torch
    cfg = synth.get_config("C5")
    with daxm.create(synth.geometry(cfg), device=0) as plan:
        st = plan.stats()
        assert (st["lock_tiles_small"] > 0) + (st["lock_tiles_large"] > 0) + (st["lock_tiles_overlap"] > 0) >= 2, st
        stack = synth.stack_torch(synth.make_maps(cfg), cfg.dtype, "cuda:0", noise=False)
        eager = torch.empty(plan.output_shape(), dtype=torch.float32, device="cuda:0")
        plan.reconstruct(stack, eager)
        graphed = torch.full_like(eager, float("nan"))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                plan.reconstruct(stack, graphed, s)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(eager, graphed)
