"""Debug aid: M = 1 / S = 2 cases, lock vs oracle, print the worst pixels."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402


def run(g, host):
    with daxm.create(g, device=0) as plan:
        st = plan.stats()
        out = plan.reconstruct(torch.from_numpy(host).cuda())
        torch.cuda.synchronize()
        return out.cpu().numpy().astype(np.float64), st


g = synth.geometry("C1")
g["depth_start"] = g["depth_end"] = 3.0
g["depth_res"] = 40.0
host = synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True)
g2 = synth.geometry("C1")
g2["wire_xyz"] = g2["wire_xyz"][[8, 12]].copy()
h2 = host[[8, 12]].copy()
for name, gg, hh in (("M=1", g, host), ("S=2", g2, h2)):
    gpu, st = run(gg, hh)
    ref = oracle.reconstruct(gg, hh)
    d = np.abs(np.diff(hh.astype(np.float64), axis=0)).sum(0)
    err = np.abs(gpu - ref) / np.maximum(d[None], 1e-300)
    print(name, "lock tiles", st["lock_tiles_small"], st["lock_tiles_large"], "max rel", err.max(), "n bad", int((err > 1e-4).sum()))
    bad = np.argwhere(err > 1e-4)[:8]
    for b in bad:
        print("  ", tuple(b), gpu[tuple(b)], ref[tuple(b)], d[tuple(b[1:])])
    if len(bad):
        b = bad[0]
        np.set_printoptions(precision=4, suppress=True, linewidth=200)
        print("gpu", gpu[:, b[1], b[2]])
        print("ref", ref[:, b[1], b[2]])
        print("series", hh[:, b[1], b[2]])
