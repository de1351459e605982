"""Run the benchmark configs through a build with DAXM_LOCK_CHECK=1 (the step-locked
kernel counts output-ring capacity violations) and print the count per config.
Usage: DAXM_LIBRARY=<lockcheck build> python scripts/lock_check.py C2 C3 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402

res = {}
for name in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    cfg = synth.get_config(name)
    for edge in cfg.edges:
        with daxm.create(synth.geometry(cfg, edge=edge), device=0) as plan:
            stack = synth.stack_torch(synth.make_maps(cfg), cfg.dtype, "cuda:0", noise=True)
            plan.reconstruct(stack)
            torch.cuda.synchronize()
            st = plan.stats()
            res[f"{name}-{edge}"] = {k: st[k] for k in ("lock_tiles_small", "lock_tiles_large", "lock_ring_violations")}
            del stack
            torch.cuda.empty_cache()
print(json.dumps(res))
