"""world > 1 kg_step on >= 2 GPUs with REAL NCCL (grouped send/recv of ids, rows and row
gradients; the dL/dtheta_D all-reduce on a split communicator; the step graph captured with the
collectives) and with the CUDA-IPC peer-memory exchange (KG_XCHG=p2p), one process per GPU under
torch.distributed.run, against the fp64 oracle of the concatenated workers (§4.1
P:L303-314).  Skipped where fewer than 2 GPUs are visible (the loopback tests,
tests/test_dist_loopback_gpu.py, cover the same path on one GPU); `bench.py --gpus N` runs the
same path for the scaling line."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("xchg", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_ranks_match_the_oracle(xchg, world):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cases = ["q2b:ip", "betae:pni", "gqe:up", "complex:1p"]
    env = dict(os.environ, KG_XCHG=xchg)
    env.pop("KG_NCCL", None)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(HERE, "_nccl_worker.py"), *cases],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok ") == len(cases), r.stdout
