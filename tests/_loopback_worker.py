"""Worker for tests/test_dist_loopback_gpu.py: world = 2 kg_step on ONE GPU, the two ranks as
threads of this process, their collectives through the library's loopback communicator
(KG_NCCL=loopback, kg_api.cu), checked against the oracle of the concatenated workers.
Every rank has its own CUDA stream, as separate processes would: the peer-memory exchange's
device-side barriers (KG_XCHG=p2p) need the ranks' kernels to run concurrently."""
import os
import sys
import threading

os.environ["KG_NCCL"] = "loopback"
# The ranks share one CUDA context here.  With lazy module loading, the first launch of a kernel
# in one rank's thread can wait for the context's running kernels -- including the other
# rank's peer-memory barrier kernel (KG_XCHG=p2p), which spins until this rank arrives.
# Separate processes (the real deployment) have separate contexts; here everything is loaded
# up front.
# Likewise the ranks' streams (six per handle, up to 4 handles) share the device's hardware work
# queues: with the default 8 connections a rank's kernel can sit in the same queue behind another
# rank's spinning barrier kernel and never start (the barrier then times out after 20 s); 32
# connections give every stream its own queue.  One rank per GPU (the deployment) never has a
# kernel of another rank on its device to wait behind.
if os.environ.get("KG_XCHG") == "p2p":     # (eager loading of torch's modules costs ~30 s)
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

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


def case(kind, structure, G=2, M=70, K=100, steps=2):
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    nid = nccl_unique_id()
    table = oracle.SparseTable(cfg, 5)
    models, errs = [None] * G, [None] * G
    barrier = threading.Barrier(G)
    for step in range(steps):
        batches = [kggen.make_batch(cfg, structure, M, K, seed=1, step=step, rank=r, mask_p=0.9) for r in range(G)]
        lr = 1e-6 if step == 0 else 1e-2          # as test_parity_gpu: step 1 tiny (H9), step 2 real
        losses = [None] * G

        def run(r):
            try:
                torch.cuda.set_device(0)
                if models[r] is None:
                    models[r] = KGModel(cfg, M, K, rank=r, world=G, nccl_id=nid, stream=torch.cuda.Stream())
                    barrier.wait()
                    models[r].init_params(5)
                    models[r].set_apply(True, stage_timing=True)   # the eager stage events too
                barrier.wait()
                losses[r] = models[r].step(models[r].host_batch(batches[r]), lr).loss
            except Exception as e:   # reported below
                errs[r] = e

        th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(120)
        assert not any(t.is_alive() for t in th), "rank thread hung"
        assert errs == [None] * G, errs
        ref = oracle.oracle_step(cfg, table, batches, lr, apply=True)
        for r in range(G):
            assert abs(losses[r] - ref.loss) <= RTOL * abs(ref.loss) + 1e-12, (step, r, losses[r], ref.loss)
        keep = np.abs(ref.m_new) >= 1e-4 * np.abs(ref.m_new).max()
        for r in range(G):      # every rank's shard rows after the owner-side update
            own = ref.uniq % G == r
            close(models[r].read_rows(ref.uniq[own]), ref.rows_new[own], f"{kind} {structure} rank {r} rows",
                  keep[own])
        dense = [m.read_dense(0) for m in models]
        assert all(np.array_equal(dense[0], x) for x in dense[1:]), "theta_D differs between ranks"
        keepd = np.abs(ref.dense_m_new) >= 1e-4 * np.abs(ref.dense_m_new).max()
        close(dense[0], ref.dense_new, f"{kind} {structure} theta_D", keepd)
    for m in models:
        m.close()
    print("ok", kind, structure, G, flush=True)


def overflow_case(G=4, M=200, K=100):
    """Distinct ids that all belong to one owner overflow its fixed-capacity bucket: every rank's
    kg_step fails with the bucket-overflow error and no table changes (transactional)."""
    cfg = kggen.ModelConfig("q2b", 40, 40000, 7)
    nid = nccl_unique_id()
    models, errs, before = [None] * G, [None] * G, [None] * G
    barrier = threading.Barrier(G)
    b = kggen.make_batch(cfg, "3i", M, K, seed=1, step=0, mask_p=0.9)
    ids = 4 * np.arange(M * 3 + M + K, dtype=np.int64)          # all owned by rank 0, all distinct
    b["anchors"] = ids[:3 * M].reshape(M, 3)
    b["answers"] = ids[3 * M:4 * M]
    b["negatives"] = ids[4 * M:]

    def run(r):
        try:
            torch.cuda.set_device(0)
            models[r] = KGModel(cfg, M, K, rank=r, world=G, nccl_id=nid, stream=torch.cuda.Stream())
            barrier.wait()
            models[r].init_params(5)
            models[r].set_apply(True)
            own = ids[ids % G == r][:64]
            before[r] = (own, models[r].read_rows(own) if len(own) else None, models[r].read_dense(0))
            barrier.wait()
            models[r].step(models[r].host_batch(b), 0.01)
        except Exception as e:
            errs[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    assert all(e is not None and "overflow" in str(e) for e in errs), errs
    for r in range(G):
        own, rows, dense = before[r]
        if rows is not None:
            assert np.array_equal(models[r].read_rows(own), rows)
        assert np.array_equal(models[r].read_dense(0), dense)
        models[r].close()
    print("ok overflow", G, flush=True)


def collective_case(kind, structure, G=2):
    """kg_score / kg_eval / kg_gather_rows with world = G (rows fetched from their owners) are
    bit-identical to one rank holding the whole table (same init, same kernels, same inputs)."""
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    nid = nccl_unique_id()
    torch.cuda.set_device(0)
    one = KGModel(cfg, 70, 100, max_cand=90)
    one.init_params(5)
    models, outs, errs = [None] * G, [None] * G, [None] * G
    barrier = threading.Barrier(G)
    ins = []
    for r in range(G):
        rng = np.random.default_rng(40 + r)
        b = kggen.make_batch(cfg, structure, 70 - 9 * r, 100, seed=3, rank=r)
        cand = rng.integers(0, 300, size=90 - 17 * r)
        M = int(b["M"])
        counts = rng.integers(1, 4, size=M)
        ans_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        ans_ids = rng.integers(0, 300, size=int(ans_off[-1]))
        negs = rng.integers(0, 300, size=(M, 50))
        ids = rng.integers(0, 300, size=0 if r == 1 else 33)          # rank 1 asks for nothing
        ins.append((b, cand, ans_off, ans_ids, negs, ids))

    def run(r):
        try:
            torch.cuda.set_device(0)
            models[r] = KGModel(cfg, 70, 100, max_cand=90, rank=r, world=G, nccl_id=nid,
                                 stream=torch.cuda.Stream())
            barrier.wait()
            models[r].init_params(5)
            barrier.wait()
            b, cand, ans_off, ans_ids, negs, ids = ins[r]
            hb = models[r].host_batch(b)
            outs[r] = (models[r].score(hb, cand), models[r].eval(hb, ans_off, ans_ids, negs),
                       models[r].gather_rows(ids), models[r].gather_rows(ids, which=2))
        except Exception as e:   # reported below
            errs[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    assert errs == [None] * G, errs
    for r in range(G):
        b, cand, ans_off, ans_ids, negs, ids = ins[r]
        hb = one.host_batch(b)
        score, (ranks, metrics), rows, vrows = outs[r]
        assert np.array_equal(score, one.score(hb, cand)), f"{kind} {structure} rank {r} kg_score"
        ranks1, metrics1 = one.eval(hb, ans_off, ans_ids, negs)
        assert np.array_equal(ranks, ranks1) and np.array_equal(metrics, metrics1), f"rank {r} kg_eval"
        assert np.array_equal(rows, one.read_rows(ids)), f"rank {r} kg_gather_rows"
        assert np.array_equal(vrows, one.read_rows(ids, which=2)), f"rank {r} kg_gather_rows (v)"
    for m in models + [one]:
        m.close()
    print("ok collective", kind, structure, G, flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        if arg == "overflow":
            overflow_case()
            continue
        parts = arg.split(":")
        if parts[0] == "collective":
            collective_case(parts[1], parts[2], G=int(parts[3]) if len(parts) > 3 else 2)
            continue
        case(parts[0], parts[1], G=int(parts[2]) if len(parts) > 2 else 2)
