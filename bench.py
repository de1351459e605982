#!/usr/bin/env python
"""Benchmark: wire-scan depth reconstruction on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one daxm_reconstruct of the whole synthetic stack of the config
(SURVEY.md §8(a) rows 3-6 in one kernel launch; the geometry pre-pass, row 2,
is per plan and timed separately as `prepass_ms`).  For N > 1 (torchrun, one
process per GPU, NCCL) every rank reconstructs its own detector row band --
no data-path collective; the timed region is bracketed by a
barrier + synchronize and the per-step time is the max over ranks.

Inputs (13.4 GB per step at C4: 6.7 GB stack read + 6.7 GB output written)
are far larger than the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "pixel·wire-steps/s"
L2_BYTES = 126 * 1024 * 1024


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(p))["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def workload_config(cfg, noise, world, parallelism_rows, edge="leading"):
    return {
        "workload": f"{cfg.name}: {cfg.description}",
        "detector": f"{cfg.n}x{cfg.n}", "n_steps": cfg.n_steps, "n_bins": cfg.n_bins,
        "depth_res_um": cfg.depth_res, "input_dtype": cfg.dtype, "edge": edge, "pixel_model": "finite",
        "stack_noise": noise, "geometry": "34-ID-E-like synthetic (SURVEY.md §8(d))",
        "parallelism": f"row-sharded x{world} (no collective)", "rows_per_gpu": parallelism_rows,
        "l2": "inputs larger than L2 (stack + output per step >> 126 MB); no flush",
    }


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_rate(cfg, maps, g, noise, budget_s, max_pixels=1 << 20, keep=4096):
    """Time the fp64 oracle (as it stands) on a random pixel sample of the workload.

    Returns the all-thread rate and its sample, the single-thread rate, and the first
    `keep` sampled pixels with their oracle outputs (for the parity spot check)."""
    import numpy as np

    import oracle
    import synth
    rng = np.random.default_rng(12345)
    threads = oracle.max_threads()
    kept = {}

    def run(n, nt=threads):
        js = rng.integers(0, cfg.n, n)
        is_ = rng.integers(0, cfg.n, n)
        ser = synth.pixel_series(maps, js, is_, cfg.dtype, noise=noise)
        t0 = time.perf_counter()
        o = oracle.reconstruct_pixels(g, js, is_, ser, n_threads=nt)
        dt = time.perf_counter() - t0
        kept.update(js=js[:keep], is_=is_[:keep], out=o[:keep].copy(), ser=ser[:keep].copy())
        return dt

    n = 256
    t = run(n)
    while t < 0.5 and n < max_pixels:
        n *= 4
        t = run(n)
    n1 = max(64, int(n * 0.1 * min(budget_s, 20.0) / max(t * threads, 1e-6)))  # ~10 % of the budget
    t1 = run(n1, 1)
    single = n1 * cfg.n_steps / t1
    n = int(min(max_pixels, max(n, n * budget_s / max(t, 1e-6))))
    t = run(n)
    return n * cfg.n_steps / t, n, t, threads, single, kept


def run_reference(args):
    """--impl reference: the fp64 CPU oracle (as it stands) on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth
    oracle.build()
    cfg = synth.get_config(args.config)
    noise = not cfg.sparse if args.noise is None else args.noise
    g = synth.geometry(cfg, edge=args.edge)
    maps = synth.make_maps(cfg)
    rng = np.random.default_rng(99)
    threads = oracle.max_threads()
    # size each step to ~args.ref_step_s of CPU work
    n = 512
    while True:
        js, is_ = rng.integers(0, cfg.n, n), rng.integers(0, cfg.n, n)
        ser = synth.pixel_series(maps, js, is_, cfg.dtype, noise=noise)
        t0 = time.perf_counter()
        oracle.reconstruct_pixels(g, js, is_, ser, n_threads=threads)
        t = time.perf_counter() - t0
        if t > 0.3 or n >= 1 << 20:
            break
        n *= 4
    n = int(max(256, min(1 << 20, n * args.ref_step_s / max(t, 1e-6))))
    times = []
    for s in range(args.warmup + args.steps):
        js, is_ = rng.integers(0, cfg.n, n), rng.integers(0, cfg.n, n)
        ser = synth.pixel_series(maps, js, is_, cfg.dtype, noise=noise)
        t0 = time.perf_counter()
        oracle.reconstruct_pixels(g, js, is_, ser, n_threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    step_s = sum(times) / len(times)
    value = n * cfg.n_steps / step_s
    sample = f"{n} random pixels x {cfg.n_steps} steps of {cfg.name} per step (fp64 oracle, all host threads)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, noise, 1, cfg.n, args.edge),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--noise", type=int, default=None, help="stack noise (default: on, except the sparse C5)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=3.0)
    ap.add_argument("--all-gather", action="store_true", help="also time an all-gather of the output planes")
    ap.add_argument("--check-gather", action="store_true",
                    help="(N>1) rank 0 compares the gathered image set bit for bit with a single-plan run of "
                         "the whole detector on its own GPU")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend for N>1 (gloo lets several ranks share one GPU)")
    ap.add_argument("--dtype", choices=["u16", "f32"], default=None,
                    help="override the config's stack dtype (e.g. C5 in fp32, SURVEY §8(d))")
    ap.add_argument("--edge", choices=["leading", "trailing", "both"], default="leading",
                    help="wire edge(s): both = leading on the decreases + trailing on the increases (R16)")
    ap.add_argument("--host-budget", type=float, default=0.0,
                    help="e2e leg out of core: cap the device memory of daxm_reconstruct_host at this many GB "
                         "(daxm_set_host_budget; 0 = whole stack resident)")
    ap.add_argument("--jitter", type=float, default=0.0,
                    help="non-straight scan (SURVEY f4): wire positions jittered by up to +-JITTER um "
                         "(exact per-step depth table + the general kernel)")
    ap.add_argument("--fraction", type=float, default=1.0,
                    help="pixel percentage (P:L299-303): reconstruct only this fraction of the pixels, the "
                         "brightest by first-step intensity (daxm_select_cutoff + daxm_set_cutoff)")
    args = ap.parse_args()
    if args.noise is not None:
        args.noise = bool(args.noise)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_13309_b200 as daxm
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    n_dev = torch.cuda.device_count()
    if world > n_dev and args.backend == "nccl":
        raise SystemExit(f"{world} ranks on {n_dev} GPU(s): NCCL needs one GPU per rank (use --backend gloo)")
    local = local % max(n_dev, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    cfg = synth.get_config(args.config)
    if args.dtype:
        import dataclasses
        cfg = dataclasses.replace(cfg, dtype=args.dtype)
    noise = (not cfg.sparse) if args.noise is None else args.noise
    g = synth.geometry(cfg, edge=args.edge)
    if args.jitter > 0:
        g["wire_xyz"] = synth.jittered_wire_positions(cfg.n_steps, t_range=cfg.t_range, amp_um=args.jitter)
    R = cfg.n
    from paper_2201_13309_b200 import multi
    r0, r1 = multi.my_band(rank, world, R)  # tile-aligned row band
    maps = synth.make_maps(cfg)
    stack = synth.stack_torch(maps, cfg.dtype, dev, noise=noise, rows=(r0, r1))
    plan = daxm.create(g, device=local, rows=(r0, r1))
    st = plan.stats()
    out = torch.empty(plan.output_shape(), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    b_in = 2 if cfg.dtype == "u16" else 4
    cutoff = None
    active = 1.0
    if args.fraction < 1.0:
        cutoff = multi.select_cutoff(plan, stack, args.fraction, R, cfg.n, stream=stream)  # global over bands
        plan.set_cutoff(cutoff)
        active = float((stack[0].float() >= float(cutoff)).double().mean())

    # warm-up
    for _ in range(args.warmup):
        plan.reconstruct(stack, out, stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t_start.record(stream)
        for s in range(K):
            ev[s][0].record(stream)
            plan.reconstruct(stack, out, stream)
            ev[s][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    kern_avg = sum(kern_ms) / len(kern_ms)
    kern_median = sorted(kern_ms)[len(kern_ms) // 2]
    # with a cutoff the input term is scaled by the active-pixel fraction (an estimate: the
    # active pixels' windows are not counted individually)
    # both edges: each edge's pass reads its windows (the stats sum the two plans'); the output is
    # stored by the first pass and read + written by the second's reduce-add
    out_passes = 3 if args.edge == "both" else 1
    alg_bytes = (active * (st["contrib_pairs"] + st["contrib_pixels"]) * b_in +
                 out_passes * st["rows"] * st["cols"] * st["n_bins"] * 4)
    achieved = alg_bytes / (kern_avg * 1e-3) / 1e9
    ms_step = total_ms / K
    ms_step_max, kern_max, achieved_min = multi.max_over_ranks([ms_step, kern_avg, -achieved], device=dev)
    achieved_min = -achieved_min
    units = R * cfg.n * cfg.n_steps
    value = units / (ms_step_max * 1e-3)

    # optional all-gather of the output planes (timed separately, not in value)
    allgather_ms = None
    gather_check = None
    if (args.all_gather or args.check_gather) and world > 1:
        bands = multi.row_bands(world, R)
        full = multi.gather_rows(out, bands)  # warm
        del full
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        a.record(stream)
        full = multi.gather_rows(out, bands)
        b.record(stream)
        torch.cuda.synchronize(dev)
        allgather_ms = multi.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        if args.check_gather and rank == 0:
            gather_check = check_gather(daxm, g, full, maps, cfg, noise, dev, stream, cutoff)
        del full
        torch.cuda.empty_cache()
        dist.barrier()

    # end to end through the C ABI from pinned host buffers (copies inside the timed region)
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, K // 4)
    if e2e_steps <= 0:
        return finish(args, rank, world, plan, cfg, g, maps, noise, K, ms_step_max, kern_max, achieved_min, value,
                      units, st, clocks, r0, r1, alg_bytes, allgather_ms, None, (cutoff, active), out,
                      kern_median, gather_check)
    h_stack = stack.cpu().pin_memory()
    h_out = torch.empty(plan.output_shape(), dtype=torch.float32).pin_memory()
    del stack
    torch.cuda.empty_cache()
    pcie = measure_pcie(dev, stream)
    if args.host_budget > 0:
        plan.set_host_budget(int(args.host_budget * 1e9))
    plan.reconstruct_host(h_stack, h_out, stream)  # warm (allocates the plan's device buffers)
    ring = plan.host_ring_info()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_a.record(stream)
    for _ in range(e2e_steps):
        plan.reconstruct_host(h_stack, h_out, stream)
    e_b.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e2e_ms = multi.max_over_ranks([e_a.elapsed_time(e_b) / e2e_steps], device=dev)[0]
    e2e_value = units / (e2e_ms * 1e-3)
    h2d = h_stack.numel() * h_stack.element_size() * world
    d2h = h_out.numel() * h_out.element_size() * world
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_ms, "path": "daxm_reconstruct_host, pinned host buffers" +
           (f", out of core: {ring['n_bands']} bands of {ring['band_rows']} rows in a {ring['ring_bytes'] / 1e9:.2f} GB "
            f"device ring" if ring["n_bands"] else ", whole stack resident")}
    if pcie:
        # PCIe roofline: the copies of both directions overlap (full duplex), so the bound is the
        # slower direction's bytes / its measured pinned-copy bandwidth
        bound_ms = max(h2d / world / (pcie["h2d_gbs"] * 1e9), d2h / world / (pcie["d2h_gbs"] * 1e9)) * 1e3
        e2e["pcie_roofline"] = dict(pcie, bound_ms=bound_ms, frac=bound_ms / e2e_ms)
    return finish(args, rank, world, plan, cfg, g, maps, noise, K, ms_step_max, kern_max, achieved_min, value,
                  units, st, clocks, r0, r1, alg_bytes, allgather_ms, e2e, (cutoff, active), out,
                  kern_median, gather_check)


def launches_per_step(st, dtype, cutoff=False):
    """Kernels one daxm_reconstruct launches (csrc/deposit.cu launch_deposit): the step-locked
    kernel once per output-ring class in use, deposit_fast (separated + dual-walk launches) if
    any non-general tile is left to it, the general kernel if any tile needs it; with a cutoff
    also tile_live and zero_dead_tiles (csrc/select.cu)."""
    if st.get("row_path"):  # row-segment path: one launch per non-empty class, cutoff in-kernel
        return int(st["row_launches"])
    general = st["general_tiles_u16" if dtype == "u16" else "general_tiles_f32"]
    small, large = st.get("lock_tiles_small", 0), st.get("lock_tiles_large", 0)
    ov = st.get("lock_tiles_overlap", 0)  # one launch per ring class in use (counted together: an upper bound)
    rest = st["n_tiles"] - general - small - large - ov
    n = (small > 0) + (large > 0) + (general > 0) + (ov > 0)
    if rest > 0:
        n += 1 + (st["overlap_tiles"] > 0)
    return int(n) + (2 if cutoff else 0)


def check_gather(daxm, g, full, maps, cfg, noise, dev, stream, cutoff):
    """--check-gather: the all-gathered image set vs one plan over the whole detector on this
    GPU (same kernels, same tiles: the row bands are tile aligned), compared bit for bit."""
    import torch

    import synth
    stack = synth.stack_torch(maps, cfg.dtype, dev, noise=noise)
    with daxm.create(g, device=dev.index) as plan:
        if cutoff is not None:
            plan.set_cutoff(cutoff)
        ref = plan.reconstruct(stack, None, stream)
        torch.cuda.synchronize(dev)
    del stack
    same = bool(torch.equal(ref.view(torch.int32), full.view(torch.int32)))
    n_diff = int((ref.view(torch.int32) != full.view(torch.int32)).sum().item())
    del ref
    return {"bitexact": same, "differing_words": n_diff, "shape": list(full.shape),
            "what": "all-gathered row bands vs a single plan of the whole detector"}


def measure_pcie(dev, stream, nbytes=1 << 30):
    """Pinned host <-> device copy bandwidth (GB/s) of this box, one direction at a time (1 GiB, best of 3)."""
    import torch
    try:
        h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        res = {}
        for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
            best = None
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                dst.copy_(src, non_blocking=True)
                b.record(stream)
                torch.cuda.synchronize(dev)
                ms = a.elapsed_time(b)
                best = ms if best is None else min(best, ms)
            res[name] = nbytes / (best * 1e-3) / 1e9
        del h, d
        torch.cuda.empty_cache()
        return res
    except Exception:
        return None


def parity_spot_check(out, kept, r0, cut):
    """After timing, compare the timed output buffer with the oracle outputs the CPU-baseline
    leg computed for its pixel sample (north_star tolerance: per bin 1e-4 * sum|dI|).  Under an
    intensity cutoff the oracle's output is zeroed at the pixels reading R14 leaves inactive
    (float32 I_0 < cutoff, oracle.active_pixels)."""
    import numpy as np
    import torch

    import oracle
    if out is None or not kept:
        return None
    js = kept["js"] - r0
    ok = (js >= 0) & (js < out.shape[1])
    js, is_ = js[ok], kept["is_"][ok]
    gpu = out[:, torch.from_numpy(js).to(out.device), torch.from_numpy(is_).to(out.device)].double().cpu().numpy().T
    ref = kept["out"][ok].copy()
    n_active = None
    if cut[0] is not None:
        act = oracle.active_pixels(kept["ser"][ok][:, 0], cut[0])
        ref[~act] = 0.0
        n_active = int(act.sum())
    ser = kept["ser"][ok].astype(np.float64)
    d = np.abs(np.diff(ser, axis=1)).sum(axis=1)
    err = np.abs(gpu - ref).max(axis=1) / np.maximum(d, 1e-300)
    err = np.where(d > 0, err, np.abs(gpu - ref).max(axis=1))
    r = {"pixels": int(len(js)), "max_bin_err_over_sum_abs_dI": float(err.max()), "tol": 1e-4,
         "pass": bool(err.max() <= 1e-4), "what": "timed output buffer vs fp64 oracle at the CPU-baseline sample"}
    if n_active is not None:
        r["active_pixels_in_sample"] = n_active
    return r


def finish(args, rank, world, plan, cfg, g, maps, noise, K, ms_step_max, kern_max, achieved_min, value, units, st,
           clocks, r0, r1, alg_bytes, allgather_ms, e2e, cut=(None, 1.0), out=None, kern_median=None,
           gather_check=None):
    import torch.distributed as dist
    if rank == 0:
        peak, peak_src = peak_hbm()
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                tj = json.load(open(prof))
                key = f"{cfg.name}:{world}"
                if key in tj:
                    traffic = tj[key]["dram_bytes_per_launch"]
            except Exception:
                traffic = None
        cpu = None
        parity = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                rate, n_pix, t_s, cores, single, kept = cpu_oracle_rate(cfg, maps, g, noise, args.cpu_budget_s)
                cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                       "sample": f"{n_pix} random pixels x {cfg.n_steps} steps of {cfg.name} ({t_s:.1f} s, fp64 "
                                 f"C oracle, OpenMP over pixels)",
                       "single_thread_value": single, "cpu_model": cpu_model()}
                parity = parity_spot_check(out, kept, r0, cut)
            except Exception as e:  # reported, not fatal
                cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(cfg, noise, world, r1 - r0, args.edge),
                           **({"wire_path": f"jittered +-{args.jitter} um (exact per-step depth table, general kernel)"}
                              if args.jitter > 0 else {})),
            "roofline": {"bound": "hbm", "achieved": achieved_min, "peak": peak, "unit": "GB/s",
                         "frac": achieved_min / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "deposit (daxm_reconstruct)", "kernel_ms": kern_max,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "bytes_rule": "sum_p (S_c(p)+1)*b_in + rows*C*M*4 (SURVEY.md §8(d))" +
                                       (" per edge, output x3 (store, then reduce-add read + write)"
                                        if args.edge == "both" else "")},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": K * world * launches_per_step(st, cfg.dtype, cut[0] is not None),
            "clocks": clocks.summary(),
            "prepass_ms": st["prepass_ms"],
            "plan": {"contrib_pairs": st["contrib_pairs"], "window_pairs": st["window_pairs"],
                     "row_path": st["row_path"], "row_tiles_small": st["row_tiles_small"],
                     "row_tiles_large": st["row_tiles_large"], "row_tiles_gen": st["row_tiles_gen"],
                     "row_tiles_general": st["row_tiles_general"],
                     "general_tiles": st["general_tiles_u16" if cfg.dtype == "u16" else "general_tiles_f32"],
                     "n_tiles": st["n_tiles"], "lock_tiles_small": st.get("lock_tiles_small"),
                     "lock_tiles_large": st.get("lock_tiles_large"), "lock_tiles_overlap": st.get("lock_tiles_overlap"),
                     "overlap_tiles": st["overlap_tiles"],
                     "staged_steps": st["staged_steps"], "fit_max_err_bins": st["fit_max_err_bins"],
                     "fit_model_err_bins": st["fit_model_err_bins"]},
        }
        if parity is not None:
            line["parity_sample"] = parity
        if kern_median is not None:
            line["roofline"]["kernel_ms_median"] = kern_median
        if cut[0] is not None:
            line["config"]["pixel_fraction"] = args.fraction
            line["config"]["cutoff_first_step_intensity"] = cut[0]
            line["config"]["active_pixels"] = cut[1]
            # the processed work: active pixels x wire steps per second (value counts every pixel)
            line["active_rate"] = {"value": value * cut[1], "unit": UNIT,
                                   "what": "value x active-pixel fraction (pixels the cutoff processes)"}
            line["roofline"]["bytes_rule"] += " with the input term x active-pixel fraction (estimate)"
        if allgather_ms is not None:
            line["all_gather_ms"] = allgather_ms
        if world > 1:
            line["config"]["backend"] = args.backend
        if gather_check is not None:
            line["gather_check"] = gather_check
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
