import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_13309_b200 as daxm, synth
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 96
g = synth.geometry("C2", n_rows=rows, n_cols=64)
g["wire_xyz"] = synth.wire_positions(1601, t_range=(40.0, 1040.0))
g["depth_res"] = 0.5
rng = np.random.default_rng(17)
host = (3000 + rng.integers(-400, 400, (1601, rows, 64))).astype(np.uint16)
plan = daxm.create(g, device=0)
print(plan.stats(), flush=True)
st = torch.from_numpy(host).cuda()
t = time.time()
out = plan.reconstruct(st)
torch.cuda.synchronize()
print("done", time.time() - t, float(out.abs().sum()), flush=True)
