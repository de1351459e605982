"""Row-sharded path with two ranks on cuda:0.

bench.py is launched by torchrun as the driver launches it for N>1, with the gloo backend
so that both ranks can share the single GPU of a gpurun box (NCCL refuses two ranks on one
device).  Each rank reconstructs its tile-aligned row band with its own plan; rank 0
all-gathers the bands and compares the image set bit for bit with one plan over the whole
detector (bench.py --check-gather).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [[], ["--fraction", "0.25"]])
def test_two_ranks_gather_bitexact(extra):
    from paper_2201_13309_b200 import _build
    _build.build_library()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--config", "C3",
           "--steps", "3", "--warmup", "3", "--check-gather", "--no-cpu-baseline", "--e2e-steps", "2"] + extra
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["backend"] == "gloo"
    assert line["config"]["rows_per_gpu"] == 512
    gc = line["gather_check"]
    assert gc["bitexact"], gc
    assert gc["shape"] == [201, 1024, 1024]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
