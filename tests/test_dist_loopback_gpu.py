"""The world > 1 training step (kg_api.cu step_dist, k_dist.cu routing kernels) on the GPU:
two ranks as threads of one process on one B200, their NCCL calls served by the library's
loopback communicator (KG_NCCL=loopback: the same buffers exchanged with device copies, rank-
order reductions) -- the pool has one GPU and NCCL refuses two ranks per device.  Checked
against the fp64 oracle of the concatenated workers (reading A18) over two steps: the loss
on every rank, every owner's updated rows, and theta_D (bitwise equal on both ranks)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("buckets,overlap,xchg", [("1", "1", "nccl"), ("0", "1", "nccl"), ("1", "0", "nccl"),
                                                  ("1", "1", "p2p")])
def test_ranks_match_the_oracle(buckets, overlap, xchg):
    """buckets = 1: fixed-capacity exchange (the default, no host round trip); 0: exact counts.
    overlap = 1 (default): the dL/dtheta_D all-reduce + dense Adam on a second stream and
    communicator, concurrent with the row-gradient exchange; 0: serial.  xchg = p2p: the row
    exchange over peer memory (one-sided reads of the owners' shards, gradient rows written into
    the owners' receive buckets, flag barriers), no NCCL call for rows."""
    cases = ["q2b:ip", "gqe:up", "betae:pni", "betae:3i", "complex:1p", "q2b:3p", "distmult-m:pi",
             "q2b:2i:4", "betae:ip:4"]
    r = subprocess.run([sys.executable, os.path.join(HERE, "_loopback_worker.py"), *cases],
                       capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, KG_DIST_BUCKETS=buckets, KG_DIST_OVERLAP=overlap, KG_XCHG=xchg))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok ") == len(cases), r.stdout


@pytest.mark.parametrize("xchg", ["nccl", "p2p"])
def test_bucket_overflow_is_reported_and_transactional(xchg):
    """Fixed-capacity buckets: distinct ids concentrated on one owner beyond its capacity make
    every rank's kg_step fail with the overflow error, and no table changes."""
    r = subprocess.run([sys.executable, os.path.join(HERE, "_loopback_worker.py"), "overflow"],
                       capture_output=True, text=True, timeout=300, env=dict(os.environ, KG_XCHG=xchg))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok overflow" in r.stdout, r.stdout


def test_collective_score_eval_gather_match_one_rank():
    """kg_score / kg_eval / kg_gather_rows at world = 2 and 3 (each rank its own queries,
    candidates and ids, of different sizes; one rank asks for no rows) equal, bit for bit, the
    same calls on one rank holding the whole table."""
    cases = ["collective:q2b:ip", "collective:betae:pni", "collective:complex:1p", "collective:gqe:up:3",
             "collective:rotate-m:pi"]
    r = subprocess.run([sys.executable, os.path.join(HERE, "_loopback_worker.py"), *cases],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok collective") == len(cases), r.stdout
