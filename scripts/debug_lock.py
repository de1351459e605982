"""Run one small reconstruction through the step-locked kernel (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
g = synth.geometry(name)
host = synth.stack_numpy(synth.make_maps(name), dtype, noise=True)
with daxm.create(g, device=0) as plan:
    print(plan.stats())
    st = torch.from_numpy(host).cuda()
    out = plan.reconstruct(st)
    torch.cuda.synchronize()
    print("ok", float(out.abs().sum()), plan.stats()["lock_ring_violations"])
