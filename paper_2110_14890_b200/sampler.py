"""ctypes binding of include/kg_sample.h (argument marshalling only).

The online sampler is native host code in libkgsample.so: reverse
directional sampling, the App. C node-cut plan, bidirectional rejection sampling and a
threaded prefetch pipeline.  Importing this module without the built library raises
ImportError; nothing here samples, traverses or verifies in Python.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SAMPLER_LIB_PATH = os.path.join(_HERE, "libkgsample.so")
if not os.path.exists(SAMPLER_LIB_PATH):
    raise ImportError(f"{SAMPLER_LIB_PATH} is missing: build it with `python paper_2110_14890_b200/build.py`")
_lib = C.CDLL(SAMPLER_LIB_PATH)

KGS_STATUS = {0: "KGS_OK", 1: "KGS_EINVAL", 2: "KGS_ENOMEM", 3: "KGS_EEXHAUSTED", 4: "KGS_ESTATE"}
STRUCTS = {"1p": 0, "2p": 1, "3p": 2, "2i": 3, "3i": 4, "ip": 5, "pi": 6, "2u": 7, "up": 8,
           "2in": 9, "3in": 10, "inp": 11, "pin": 12, "pni": 13}
STRUCT_NAME = {v: k for k, v in STRUCTS.items()}
N_ANCHORS = [1, 1, 1, 2, 3, 2, 2, 2, 2, 2, 3, 2, 2, 2]
N_RELS = [1, 2, 3, 2, 3, 3, 3, 2, 3, 2, 3, 3, 3, 3]

_P = C.c_void_p
_sig = {
    "kgs_graph_create": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, _P, _P, _P, C.c_int32, C.POINTER(_P)]),
    "kgs_graph_destroy": (None, [_P]),
    "kgs_graph_edges": (C.c_int64, [_P]),
    "kgs_graph_roots": (C.c_int64, [_P]),
    "kgs_plan": (C.c_int, [C.c_int32, _P, _P, _P, _P, _P]),
    "kgs_sample": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int64, C.c_int32, C.c_int32,
                             _P, _P, _P, _P, _P, _P]),
    "kgs_verify": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.c_int32, _P, C.c_int32, _P, C.c_int32]),
    "kgs_answers": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, C.c_int64, C.c_int32]),
    "kgs_pipeline_create": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int64,
                                      C.c_int32, C.c_int32, C.POINTER(_P)]),
    "kgs_pipeline_next": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "kgs_pipeline_destroy": (None, [_P]),
    "kgs_last_error": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args
    globals()[_name] = _f

SAMPLER_EXPORTED = sorted(_sig)


class KGSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{KGS_STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st):
    if st != 0:
        raise KGSError(st, kgs_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data


def plan(structure: str):
    """(u, s, o, cut node ids) of the App. C plan of a structure (preorder node ids)."""
    n = C.c_int32()
    u, s, o, cut = (np.zeros(16, np.int32) for _ in range(4))
    _check(kgs_plan(STRUCTS[structure], C.byref(n), _p(u), _p(s), _p(o), _p(cut)))
    k = n.value
    return u[:k].tolist(), s[:k].tolist(), o[:k].tolist(), np.nonzero(cut[:k])[0].tolist()


class KGSampler:
    """Owner of one native graph (CSR indices of a KG's triples)."""

    def __init__(self, kg: dict, n_threads: int = None):
        self.n_threads = n_threads or os.cpu_count() or 1
        self.V, self.R = int(kg["n_entities"]), int(kg["n_relations"])
        h = np.ascontiguousarray(kg["h"], np.int64)
        r = np.ascontiguousarray(kg["r"], np.int32)
        t = np.ascontiguousarray(kg["t"], np.int64)
        self.g = _P()
        _check(kgs_graph_create(self.V, self.R, len(h), _p(h), _p(r), _p(t), self.n_threads, C.byref(self.g)))
        self.n_edges = kgs_graph_edges(self.g)
        self.n_roots = kgs_graph_roots(self.g)

    def sample(self, structure: str, M: int, K: int, seed: int = 0, step: int = 0, rank: int = 0,
               n_threads: int = None) -> dict:
        """One batch in the kggen.make_batch / kg_step format (+ attempts per query)."""
        sid = STRUCTS[structure]
        out = dict(structure=structure, M=M, K=K,
                   anchors=np.zeros((M, N_ANCHORS[sid]), np.int64), relations=np.zeros((M, N_RELS[sid]), np.int32),
                   answers=np.zeros(M, np.int64), negatives=np.zeros(max(K, 1), np.int64)[:K],
                   mask=np.zeros((M, max(1, (K + 31) // 32)), np.uint32)[:, :(K + 31) // 32],
                   attempts=np.zeros(M, np.int32))
        out["negatives"] = np.ascontiguousarray(out["negatives"])
        out["mask"] = np.ascontiguousarray(out["mask"])
        _check(kgs_sample(self.g, sid, M, K, seed, step, rank, n_threads or self.n_threads,
                          _p(out["anchors"]), _p(out["relations"]), _p(out["answers"]), _p(out["negatives"]),
                          _p(out["mask"]), _p(out["attempts"])))
        return out

    def verify(self, structure: str, anchors, relations, cand, shared: bool = True, n_threads: int = None):
        """bool [M, n_cand]: cand is an answer of query i (exact, bidirectional search)."""
        sid = STRUCTS[structure]
        a = np.ascontiguousarray(anchors, np.int64).reshape(-1, N_ANCHORS[sid])
        r = np.ascontiguousarray(relations, np.int32).reshape(-1, N_RELS[sid])
        M = a.shape[0]
        c = np.ascontiguousarray(cand, np.int64)
        n = c.shape[-1]
        out = np.zeros((M, n), np.uint8)
        _check(kgs_verify(self.g, sid, M, _p(a), _p(r), n, _p(c), 1 if shared else 0, _p(out),
                          n_threads or self.n_threads))
        return out.astype(bool)

    def answers(self, structure: str, anchors, relations, n_threads: int = None):
        """Answer sets by forward traversal: (offsets int64 [M + 1], ids int64 [offsets[M]])."""
        sid = STRUCTS[structure]
        a = np.ascontiguousarray(anchors, np.int64).reshape(-1, N_ANCHORS[sid])
        r = np.ascontiguousarray(relations, np.int32).reshape(-1, N_RELS[sid])
        M = a.shape[0]
        off = np.zeros(M + 1, np.int64)
        nt = n_threads or self.n_threads
        _check(kgs_answers(self.g, sid, M, _p(a), _p(r), _p(off), None, 0, nt))
        ids = np.zeros(max(1, int(off[-1])), np.int64)
        _check(kgs_answers(self.g, sid, M, _p(a), _p(r), _p(off), _p(ids), len(ids), nt))
        return off, ids[:int(off[-1])]

    def pipeline(self, structures, M, K, seed=0, rank=0, first_step=0, depth=None, n_workers=None, pin=False):
        return Pipeline(self, structures, M, K, seed, rank, first_step, depth, n_workers, pin)

    def close(self):
        if self.g:
            kgs_graph_destroy(self.g)
            self.g = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Pipeline:
    """Threaded prefetch of the batches of consecutive steps (ring of `depth` slots).

    next() returns views into buffers it reuses; with pin=True (torch present) the
    buffers are pinned host memory, ready for kg_step's H2D copy.
    """

    def __init__(self, smp: KGSampler, structures, M, K, seed=0, rank=0, first_step=0, depth=None,
                 n_workers=None, pin=False):
        self.smp = smp
        self.M, self.K = M, K
        n_workers = n_workers or max(1, (os.cpu_count() or 2) - 1)
        depth = depth or 2 * n_workers
        self.st = np.array([STRUCTS[s] for s in structures], np.int32)
        self.p = _P()
        _check(kgs_pipeline_create(smp.g, _p(self.st), len(self.st), M, K, seed, rank, first_step, depth, n_workers,
                                   C.byref(self.p)))
        W = max(1, (K + 31) // 32)
        shapes = dict(anchors=((M, 3), np.int64), relations=((M, 3), np.int32), answers=((M,), np.int64),
                      negatives=((max(K, 1),), np.int64), mask=((M, W), np.uint32))
        if pin:   # page-locked buffers (numpy views of pinned torch tensors): kg_step's H2D is a DMA
            import torch
            tdt = {np.int64: torch.int64, np.int32: torch.int32, np.uint32: torch.int32}
            self._pinned = {k: torch.zeros(sh, dtype=tdt[dt], pin_memory=True) for k, (sh, dt) in shapes.items()}
            self.buf = {k: t.numpy().view(shapes[k][1]) for k, t in self._pinned.items()}
        else:
            self.buf = {k: np.zeros(sh, dt) for k, (sh, dt) in shapes.items()}
        self.wait_ms = 0.0

    def next(self) -> dict:
        sid, step, w = C.c_int32(), C.c_int64(), C.c_double()
        b = self.buf
        _check(kgs_pipeline_next(self.p, C.byref(sid), C.byref(step), _p(b["anchors"]), _p(b["relations"]),
                                 _p(b["answers"]), _p(b["negatives"]), _p(b["mask"]), C.byref(w)))
        self.wait_ms += w.value
        s = sid.value
        na, nr = N_ANCHORS[s], N_RELS[s]
        return dict(structure=STRUCT_NAME[s], step=step.value, M=self.M, K=self.K,
                    anchors=b["anchors"].reshape(-1)[:self.M * na].reshape(self.M, na),
                    relations=b["relations"].reshape(-1)[:self.M * nr].reshape(self.M, nr),
                    answers=b["answers"], negatives=b["negatives"][:self.K], mask=b["mask"])

    def close(self):
        if self.p:
            kgs_pipeline_destroy(self.p)
            self.p = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_eval_set(test: KGSampler, valid: KGSampler, structure: str, n_queries: int, n_neg: int = 1000,
                   seed: int = 0, step: int = 0, max_rounds: int = 16):
    """Evaluation set of App. E for kg_eval: queries grounded on G_test by reverse
    sampling, their missing answers A_q(G_test) minus A_q(G_valid) (kept: at least one), and n_neg
    negatives per query drawn uniformly from V and filtered exactly to V minus A_q(G_test) by the
    native bidirectional verification.  Traversal and verification run in libkgsample.so; the
    set differences / selection here are host bookkeeping.  Returns (batch, ans_off, ans_ids,
    negatives [M][n_neg]) with M = n_queries."""
    sid = STRUCTS[structure]
    keep_a, keep_r, hard = [], [], []
    for rnd in range(max_rounds):
        b = test.sample(structure, 2 * n_queries, 0, seed=seed, step=step * max_rounds + rnd)
        ot, it = test.answers(structure, b["anchors"], b["relations"])
        ov, iv = valid.answers(structure, b["anchors"], b["relations"])
        for i in range(2 * n_queries):
            h = np.setdiff1d(it[ot[i]:ot[i + 1]], iv[ov[i]:ov[i + 1]], assume_unique=True)
            if len(h):
                keep_a.append(b["anchors"][i])
                keep_r.append(b["relations"][i])
                hard.append(h)
            if len(hard) == n_queries:
                break
        if len(hard) == n_queries:
            break
    if len(hard) < n_queries:
        raise KGSError(3, f"only {len(hard)} of {n_queries} {structure} queries have missing answers")
    anchors = np.ascontiguousarray(np.stack(keep_a), np.int64).reshape(n_queries, N_ANCHORS[sid])
    relations = np.ascontiguousarray(np.stack(keep_r), np.int32).reshape(n_queries, N_RELS[sid])
    ans_off = np.zeros(n_queries + 1, np.int64)
    ans_off[1:] = np.cumsum([len(h) for h in hard])
    ans_ids = np.concatenate(hard).astype(np.int64)
    rng = np.random.default_rng([seed, step, sid, 0xE7A1])
    neg = np.zeros((n_queries, n_neg), np.int64)
    filled = np.zeros(n_queries, np.int64)
    for rnd in range(max_rounds):
        need = n_queries * n_neg - int(filled.sum())
        if need == 0:
            break
        cand = rng.integers(0, test.V, size=(n_queries, 2 * n_neg), dtype=np.int64)
        is_ans = test.verify(structure, anchors, relations, cand, shared=False)
        for i in range(n_queries):
            ok = cand[i][~is_ans[i]]
            take = min(len(ok), n_neg - filled[i])
            neg[i, filled[i]:filled[i] + take] = ok[:take]
            filled[i] += take
    if int(filled.sum()) < n_queries * n_neg:
        raise KGSError(3, "could not draw enough non-answers")
    batch = dict(structure=structure, M=n_queries, anchors=anchors, relations=relations)
    return batch, ans_off, ans_ids, neg
