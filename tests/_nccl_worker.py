"""Worker for tests/test_multigpu_nccl.py: one process per GPU under torch.distributed.run,
world = WORLD_SIZE ranks of kg_step over REAL NCCL (and, with KG_XCHG=p2p, CUDA-IPC peer
memory), checked on rank 0 against the fp64 oracle of the concatenated workers (reading A18):
the loss of every rank, every owner's updated rows and theta_D (bitwise equal on all ranks)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import kggen  # noqa: E402
import oracle  # noqa: E402
from paper_2110_14890_b200 import KGModel, nccl_unique_id  # noqa: E402

RTOL = 1e-5


def close(x, ref, what, mask=None):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(x - ref)
    tol = RTOL * np.abs(ref) + RTOL * np.abs(ref).max()
    bad = err > tol
    if mask is not None:
        bad &= mask
    assert not bad.any(), f"{what}: {bad.sum()}/{bad.size} out of tolerance, max err {err.max():.3g}"


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")            # host-side plumbing only; the step's collectives are NCCL
    for spec in sys.argv[1:]:
        kind, structure = spec.split(":")
        cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        gm = KGModel(cfg, 70, 100, rank=rank, world=world, nccl_id=obj[0])
        gm.init_params(5)
        gm.set_apply(True)
        table = oracle.SparseTable(cfg, 5) if rank == 0 else None
        for step in range(2):
            batches = [kggen.make_batch(cfg, structure, 70, 100, seed=1, step=step, rank=r, mask_p=0.9)
                       for r in range(world)]
            lr = 1e-6 if step == 0 else 1e-2
            loss = gm.step(gm.host_batch(batches[rank]), lr).loss
            losses = [None] * world
            dist.all_gather_object(losses, loss)
            ids = np.arange(cfg.n_entities, dtype=np.int64)
            own = ids[ids % world == rank]
            rows = [None] * world
            dist.all_gather_object(rows, (own, gm.read_rows(own)))
            dense = [None] * world
            dist.all_gather_object(dense, gm.read_dense(0))
            if rank == 0:
                ref = oracle.oracle_step(cfg, table, batches, lr, apply=True)
                for r in range(world):
                    assert abs(losses[r] - ref.loss) <= RTOL * abs(ref.loss) + 1e-12, (step, r, losses[r], ref.loss)
                allrows = np.zeros((cfg.n_entities, cfg.dim))
                for o, x in rows:
                    allrows[o] = x
                keep = np.abs(ref.m_new) >= 1e-4 * np.abs(ref.m_new).max()
                close(allrows[ref.uniq], ref.rows_new, f"{spec} rows", keep)
                assert all(np.array_equal(dense[0], x) for x in dense[1:]), "theta_D differs between ranks"
                keepd = np.abs(ref.dense_m_new) >= 1e-4 * np.abs(ref.dense_m_new).max()
                close(dense[0], ref.dense_new, f"{spec} theta_D", keepd)
        gm.close()
        if rank == 0:
            print("ok", spec, world, os.environ.get("KG_XCHG", "nccl"), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
