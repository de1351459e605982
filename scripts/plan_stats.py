"""Print plan statistics for every BASELINE config (GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    cfg = synth.get_config(name)
    for edge in cfg.edges:
        with daxm.create(synth.geometry(cfg, edge=edge), device=0) as plan:
            st = plan.stats()
        print(name, edge, json.dumps(st))
