"""One reconstruction per path on small configs, for compute-sanitizer runs
(scripts/gpu_sanitize.sh): C1 finite/point (row kernel), C2 trailing, a ragged detector
(row + general tails), C2 with a cutoff, the host path, and the general kernel.
Each result is checked against the fp64 oracle so a run that 'passes' the tool also computes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import oracle  # noqa: E402
import paper_2201_13309_b200 as daxm  # noqa: E402
import parity  # noqa: E402
import synth  # noqa: E402


def case(name, g, host, cutoff=None, host_path=False):
    with daxm.create(g, device=0) as plan:
        if cutoff is not None:
            plan.set_cutoff(cutoff)
        if host_path:
            out = plan.reconstruct_host(host)
            gpu = np.asarray(out)
        else:
            out = plan.reconstruct(torch.from_numpy(np.ascontiguousarray(host)).cuda())
            torch.cuda.synchronize()
            gpu = out.cpu().numpy()
    ref = oracle.reconstruct(g, host)
    if cutoff is not None:
        ref[:, ~oracle.active_pixels(host[0], cutoff)] = 0
    parity.check(gpu, ref, host, name)
    print("ok", name, flush=True)


which = sys.argv[1:] or ["c1", "c1p", "c2t", "ragged", "cut", "host", "both", "prof", "ooc", "general"]
if "c1" in which:
    case("C1 finite f32", synth.geometry("C1"), synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True))
if "c1p" in which:
    case("C1 point u16", synth.geometry("C1", pixel_model="point"),
         synth.stack_numpy(synth.make_maps("C1"), "u16", noise=True))
if "c2t" in which:
    case("C2 trailing", synth.geometry("C2", edge="trailing"), synth.stack_numpy(synth.make_maps("C2"), "f32", noise=True))
if "ragged" in which:
    g = synth.geometry("C2", n_rows=77, n_cols=45)
    g["wire_xyz"] = synth.wire_positions(61, t_range=(40.0, 1040.0))
    rng = np.random.default_rng(3)
    case("ragged", g, (1000 + rng.integers(-300, 300, (61, 77, 45))).astype(np.float32))
if "cut" in which:
    host = synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True)
    case("C2 cutoff", synth.geometry("C2"), host, cutoff=oracle.select_cutoff(host[0], 0.25))
if "host" in which:
    case("C2 host path", synth.geometry("C2"), synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True),
         host_path=True)
if "both" in which:  # both-edges children: clamp + red.global.add copy-out
    case("C2 both edges", synth.geometry("C2", edge="both"), synth.stack_numpy(synth.make_maps("C2"), "f32", noise=True))
if "prof" in which:  # fused depth profile (the copy-out's warp sums)
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True)
    with daxm.create(g, device=0) as plan:
        out, prof = plan.reconstruct_profile(torch.from_numpy(host).cuda())
        torch.cuda.synchronize()
        ref = oracle.reconstruct(g, host)
        parity.check(out.cpu().numpy(), ref, host, "C2 fused profile")
        assert np.allclose(prof.cpu().numpy(), oracle.depth_profile(ref), rtol=1e-5, atol=1e-3 * np.abs(ref).sum())
    print("ok C2 fused profile", flush=True)
if "ooc" in which:  # out-of-core host ring (two device slots, band plans)
    g = synth.geometry("C2")
    host = synth.stack_numpy(synth.make_maps("C2"), "u16", noise=True)
    with daxm.create(g, device=0) as plan:
        plan.set_host_budget((host.nbytes + 101 * 512 * 512 * 4) // 2)
        gpu = np.asarray(plan.reconstruct_host(host))
        assert plan.host_ring_info()["n_bands"] >= 2
    parity.check(gpu, oracle.reconstruct(g, host), host, "C2 out of core")
    print("ok C2 out of core", flush=True)
if "general" in which:
    os.environ["DAXM_FORCE_GENERAL"] = "1"
    case("C1 general", synth.geometry("C1"), synth.stack_numpy(synth.make_maps("C1"), "f32", noise=True))
torch.cuda.synchronize()
torch.cuda.empty_cache()  # leave no cached torch blocks for --leak-check (the plans freed theirs)
