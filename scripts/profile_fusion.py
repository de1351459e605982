"""Fused vs unfused depth profile: per config, CUDA-event times of
(a) daxm_reconstruct alone, (b) daxm_reconstruct + daxm_depth_profile (the output read back),
(c) daxm_reconstruct_profile (the row kernel's per-tile plane sums + a tile reduction).
Prints one JSON line per config."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2]


for name in sys.argv[1:] or ["C4", "C5"]:
    cfg = synth.get_config(name)
    g = synth.geometry(cfg)
    maps = synth.make_maps(cfg)
    stack = synth.stack_torch(maps, cfg.dtype, "cuda:0", noise=not cfg.sparse)
    with daxm.create(g, device=0) as plan:
        out = torch.empty(plan.output_shape(), dtype=torch.float32, device="cuda:0")
        prof = torch.empty(plan.n_bins, dtype=torch.float64, device="cuda:0")
        a = timed(lambda: plan.reconstruct(stack, out))
        b = timed(lambda: (plan.reconstruct(stack, out), plan.depth_profile(out, prof)))
        c = timed(lambda: plan.reconstruct_profile(stack, out, prof))
        p_only = timed(lambda: plan.depth_profile(out, prof))
        f, _ = plan.reconstruct_profile(stack, out, prof)
        fused = prof.clone()
        plan.depth_profile(out, prof)
        rel = float((fused - prof).abs().max() / prof.abs().max())
    print(json.dumps({"config": name, "reconstruct_ms": a, "reconstruct_plus_profile_ms": b,
                      "profile_kernel_ms": p_only, "fused_ms": c, "fused_overhead_ms": c - a,
                      "unfused_overhead_ms": b - a, "max_rel_diff_fused_vs_unfused": rel,
                      "output_bytes": out.numel() * 4}), flush=True)
    del stack, out
    torch.cuda.empty_cache()
