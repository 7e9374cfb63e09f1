"""The multi-rank protocol of kg_step (world > 1) on CPU with gloo, world_size 2.

kg_step with world > 1 (kg_api.cu::step_dist, k_dist.cu) row-shards theta_E
(owner(id) = id % G, local row = id // G), routes each rank's distinct ids to
their owners (stable partition by owner, ascending ids within an owner),
returns the owners' rows, sends each rank's merged row gradients (scaled by
1/(M G)) back to the owners, which sum the contributions in (source rank,
position) order; dL/dtheta_D is all-reduced; the loss is the sum of the
per-rank scaled sums (reading A18).  This test runs that protocol with
torch.distributed (gloo) around the CPU oracle and checks that it reproduces
the single-process oracle of the concatenated workers exactly (up to fp64
rounding): the rows every rank receives, the owner-merged row gradients,
the all-reduced dense gradient and the global loss.  The device kernels that
implement the same routing run only on GPUs (-m gpu).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import kggen
import oracle

G = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def owner_partition(uniq, G):
    """Mirror of owner_partition_kernel: stable partition of ascending ids by owner."""
    owners = uniq % G
    counts = np.array([(owners == o).sum() for o in range(G)])
    send_ids = np.concatenate([uniq[owners == o] for o in range(G)])
    pos = np.empty(len(uniq), np.int64)
    off = np.concatenate([[0], np.cumsum(counts)])
    for o in range(G):
        pos[owners == o] = off[o] + np.arange(counts[o])
    return send_ids, pos, counts


def exchange(send_chunks, rank, world):
    """Variable-size all-to-all with point-to-point gloo messages (sizes exchanged first)."""
    sizes = torch.tensor([c.shape[0] for c in send_chunks], dtype=torch.int64)
    all_sizes = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    tail = send_chunks[0].shape[1:]
    recv = [torch.zeros((int(all_sizes[s][rank]),) + tuple(tail), dtype=send_chunks[0].dtype) for s in range(world)]
    reqs = []
    for o in range(world):
        if o == rank:
            recv[o].copy_(send_chunks[o])
            continue
        if send_chunks[o].shape[0]:
            reqs.append(dist.isend(send_chunks[o].contiguous(), o))
        if recv[o].shape[0]:
            reqs.append(dist.irecv(recv[o], o))
    for r in reqs:
        r.wait()
    return recv


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = kggen.ModelConfig("q2b", 8, 40, 5)
        seed = 3
        batches = [kggen.make_batch(cfg, "2i", 6, 9, seed=seed, step=0, rank=r, mask_p=0.8) for r in range(world)]
        mine = batches[rank]
        # the owner's shard of theta_E (initial values; every rank owns ids with id % G == rank)
        shard_ids = np.arange(rank, cfg.n_entities, world)
        table = oracle.SparseTable(cfg, seed)
        shard = dict(zip(shard_ids.tolist(), table.get(shard_ids)[0]))
        # 1. distinct ids of this rank -> owners
        ids = np.concatenate([mine["anchors"].ravel(), mine["answers"], mine["negatives"]])
        uniq = np.array(sorted(set(ids.tolist())), np.int64)
        send_ids, pos, counts = owner_partition(uniq, world)
        off = np.concatenate([[0], np.cumsum(counts)])
        req = exchange([torch.from_numpy(send_ids[off[o]:off[o + 1]]) for o in range(world)], rank, world)
        # 2. owners return their rows in request order
        rows_back = [torch.from_numpy(np.stack([shard[int(i)] for i in r.tolist()]) if len(r) else
                                      np.zeros((0, cfg.dim), np.float32)) for r in req]
        got = exchange(rows_back, rank, world)
        Xin = torch.cat(got).numpy()
        # received rows equal the global table rows of this rank's distinct ids
        np.testing.assert_array_equal(Xin[pos], table.get(uniq)[0])
        # 3. this rank's scaled gradient contribution (its batch alone, scaled by 1/G: A18)
        local = oracle.oracle_step(cfg, oracle.SparseTable(cfg, seed), [mine], 1e-3, apply=False)
        np.testing.assert_array_equal(local.uniq, uniq)
        g_local = local.grad_rows / world
        gsend = g_local[np.argsort(pos)]                    # send order
        grads = exchange([torch.from_numpy(gsend[off[o]:off[o + 1]]) for o in range(world)], rank, world)
        # 4. owner merge in (source rank, position) order
        keys = torch.cat(req).numpy()
        gall = torch.cat(grads).numpy()
        merged = {}
        for k, g in zip(keys.tolist(), gall):
            merged[k] = merged.get(k, 0.0) + g
        # 5. dense gradient all-reduce and global loss
        gd = torch.from_numpy(local.grad_dense / world)
        dist.all_reduce(gd)
        loss = torch.tensor([local.loss / world], dtype=torch.float64)
        dist.all_reduce(loss)
        # reference: one oracle step over both workers' batches (A18)
        ref = oracle.oracle_step(cfg, oracle.SparseTable(cfg, seed), batches, 1e-3, apply=False)
        gref = dict(zip(ref.uniq.tolist(), ref.grad_rows))
        owned = [k for k in gref if k % world == rank]
        assert sorted(merged) == sorted(owned)
        for k in owned:
            np.testing.assert_allclose(merged[k], gref[k], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(gd.numpy(), ref.grad_dense, rtol=1e-12, atol=1e-15)
        assert abs(float(loss) - ref.loss) <= 1e-12 * abs(ref.loss)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_row_sharded_protocol_matches_oracle_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, q)) for r in range(G)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(G))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_owner_partition_mirror():
    uniq = np.array([0, 1, 2, 5, 7, 8, 11])
    send_ids, pos, counts = owner_partition(uniq, 3)
    assert counts.tolist() == [1, 2, 4]
    np.testing.assert_array_equal(send_ids, [0, 1, 7, 2, 5, 8, 11])
    np.testing.assert_array_equal(send_ids[pos], uniq)
