"""Row-tile admission statistics per config (GPU): classes, ring need, reject reasons."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_13309_b200 as daxm  # noqa: E402
import synth  # noqa: E402

WHY = ["mode", "kt", "input", "density", "top", "ring", "order", "iter"]
for arg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    name, _, edge = arg.partition(":")
    cfg = synth.get_config(name)
    with daxm.create(synth.geometry(cfg, edge=edge or "leading"), device=0) as plan:
        st = plan.stats()
    rej = {w: n for w, n in zip(WHY, st["row_reject"]) if n}
    print(arg, json.dumps({"small": st["row_tiles_small"], "large": st["row_tiles_large"],
                            "general": st["row_tiles_general"], "gen": st["row_tiles_gen"], "rej_gen": st["row_reject_more"],
                            "row_path": st["row_path"], "need": st["row_ring_need_max"], "reject": rej,
                            "nb_mid": st["row_tiles_nb_mid"], "kmax_hist": st["row_kmax_hist"],
                            "model_err": st["fit_model_err_bins"], "max_err": st["fit_max_err_bins"],
                            "prepass_ms": st["prepass_ms"]}), flush=True)
