"""-m gpu, needs >= 2 GPUs (gpurun --gpus 2): the multi-GPU shards with the
fused NVLink gather give cuda:0 outputs byte-identical to a
1-GPU solve of the same scenarios (tools/multi_gpu_check.py under torchrun)."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,n,prec,gather", [("C4", 200_000, 0, "chunked"), ("C4", 200_000, 0, "fused"),
                                               ("C3", 100_003, 1, "chunked")])
def test_gather_byte_identical(cfg, n, prec, gather):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    ws = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ws}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "multi_gpu_check.py"), "--config", cfg, "--scenarios", str(n),
           "--precision", str(prec), "--gather", gather]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads(lines[-1])
    assert res["ok"] and all(res["arrays_identical"].values()), res
