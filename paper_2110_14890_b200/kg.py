"""ctypes binding of include/kg.h (argument marshalling only).

Every function of the C-ABI is exposed under the same name.  There is no
fallback: importing this module without a built `libkg.so` raises ImportError,
and every compute call goes to the sm_100a kernels inside the library.
PyTorch is used by `KGModel` only to own device memory (the caller-owned
tables of kg_bind) and to name the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkg.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2110_14890_b200/build.py` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

KG_OK, KG_EINVAL, KG_EUNSUPPORTED, KG_ENOMEM, KG_ECUDA, KG_ENCCL, KG_ENONFINITE, KG_ESTATE = range(8)
STATUS = {0: "KG_OK", 1: "KG_EINVAL", 2: "KG_EUNSUPPORTED", 3: "KG_ENOMEM", 4: "KG_ECUDA",
          5: "KG_ENCCL", 6: "KG_ENONFINITE", 7: "KG_ESTATE"}
KINDS = {"gqe": 0, "q2b": 1, "betae": 2, "transe": 3, "rotate": 4, "distmult": 5, "complex": 6,
         "rotate-m": 7, "distmult-m": 8, "complex-m": 9}
STRUCTS = {"1p": 0, "2p": 1, "3p": 2, "2i": 3, "3i": 4, "ip": 5, "pi": 6, "2u": 7, "up": 8,
           "2in": 9, "3in": 10, "inp": 11, "pin": 12, "pni": 13}


class kg_config(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_int32), ("n_entities", C.c_int64),
                ("n_relations", C.c_int32), ("hidden", C.c_int32), ("gamma", C.c_float),
                ("box_alpha", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("max_M", C.c_int32), ("max_K", C.c_int32), ("max_cand", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p),
                ("score_precision", C.c_int32)]


class kg_tables(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("ent", "ent_m", "ent_v", "dense", "dense_m", "dense_v")]


class kg_batch(C.Structure):
    _fields_ = [("structure", C.c_int32), ("M", C.c_int32), ("K", C.c_int32),
                ("anchors", C.c_void_p), ("relations", C.c_void_p), ("answers", C.c_void_p),
                ("negatives", C.c_void_p), ("mask", C.c_void_p), ("on_device", C.c_int32)]


class kg_step_info(C.Structure):
    _fields_ = [("loss", C.c_double), ("n_touched", C.c_int32), ("step", C.c_int64),
                ("kernels", C.c_int32), ("gemms", C.c_int32), ("stage_ms", C.c_float * 10)]


_H = C.c_void_p
_sig = {
    "kg_create": (C.c_int, [C.POINTER(kg_config), C.POINTER(_H)]),
    "kg_shard_rows": (C.c_int64, [_H]),
    "kg_dense_size": (C.c_int64, [_H]),
    "kg_workspace_size": (C.c_int64, [_H]),
    "kg_bind": (C.c_int, [_H, C.POINTER(kg_tables), C.c_void_p]),
    "kg_init_params": (C.c_int, [_H, C.c_uint64]),
    "kg_step": (C.c_int, [_H, C.POINTER(kg_batch), C.c_float, C.POINTER(kg_step_info)]),
    "kg_sync": (C.c_int, [_H, C.POINTER(kg_step_info)]),
    "kg_result": (C.c_int, [_H, C.POINTER(kg_step_info)]),
    "kg_score": (C.c_int, [_H, C.POINTER(kg_batch), C.c_void_p, C.c_int32, C.c_void_p]),
    "kg_score_each": (C.c_int, [_H, C.POINTER(kg_batch), C.c_void_p, C.c_int32, C.c_void_p]),
    "kg_eval": (C.c_int, [_H, C.POINTER(kg_batch), C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                          C.c_void_p]),
    "kg_read_rows": (C.c_int, [_H, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "kg_gather_rows": (C.c_int, [_H, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "kg_write_rows": (C.c_int, [_H, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "kg_read_dense": (C.c_int, [_H, C.c_int32, C.c_void_p]),
    "kg_write_dense": (C.c_int, [_H, C.c_int32, C.c_void_p]),
    "kg_last_grads": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32),
                                C.c_void_p, C.c_void_p]),
    "kg_set_apply": (C.c_int, [_H, C.c_int32]),
    "kg_last_error": (C.c_char_p, [_H]),
    "kg_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "kg_get_step": (C.c_int, [_H, C.POINTER(C.c_int64)]),
    "kg_set_step": (C.c_int, [_H, C.c_int64]),
    "kg_test_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                               C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_float,
                               C.c_void_p]),
    "kg_destroy": (None, [_H]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args
    globals()[_name] = _f

EXPORTED = sorted(_sig)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be broadcast to the other ranks before kg_create."""
    buf = C.create_string_buffer(128)
    check(kg_nccl_unique_id(buf))
    return buf.raw


class KGError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status, handle=None):
    if status != KG_OK:
        msg = kg_last_error(handle).decode() if handle else ""
        raise KGError(status, msg)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()   # torch tensor (device or pinned host)


SCORE_PRECISIONS = {"fp32": 0, "bf16": 1}


def make_config(cfg, max_M, max_K, max_cand=0, rank=0, world=1, nccl_id=None, score_precision="fp32") -> kg_config:
    """kg_config from a kggen.ModelConfig-like object (kind, dim, n_entities, ...)."""
    return kg_config(KINDS[cfg.kind], cfg.dim, cfg.n_entities, cfg.n_relations, cfg.hidden or 0,
                     cfg.gamma, cfg.box_alpha, cfg.beta1, cfg.beta2, cfg.eps, max_M, max_K, max_cand,
                     rank, world, nccl_id, SCORE_PRECISIONS[score_precision])


class KGModel:
    """Convenience owner of one handle + its caller-owned tables (torch device memory)."""

    def __init__(self, cfg, max_M, max_K, max_cand=0, device="cuda", stream=None, rank=0, world=1,
                 nccl_id: bytes = None, host_tables=(), score_precision="fp32"):
        """host_tables: names among ("ent", "ent_m", "ent_v") to keep in pinned host memory
        (the host tier of kg_bind); the others live in device memory."""
        import torch
        self.cfg = cfg
        self.torch = torch
        self.h = _H()
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.conf = make_config(cfg, max_M, max_K, max_cand, rank, world,
                                C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None,
                                score_precision)
        check(kg_create(C.byref(self.conf), C.byref(self.h)))
        self.rows = kg_shard_rows(self.h)
        self.dense_size = kg_dense_size(self.h)
        self.workspace_bytes = kg_workspace_size(self.h)
        d = cfg.dim
        f32 = torch.float32
        def table(name):
            if name in host_tables:
                return torch.empty((self.rows, d), dtype=f32, pin_memory=True)
            return torch.empty((self.rows, d), dtype=f32, device=device)
        self.ent, self.ent_m, self.ent_v = table("ent"), table("ent_m"), table("ent_v")
        self.dense = torch.empty(self.dense_size, dtype=f32, device=device)
        self.dense_m = torch.empty_like(self.dense)
        self.dense_v = torch.empty_like(self.dense)
        self.tables = kg_tables(*[t.data_ptr() for t in (self.ent, self.ent_m, self.ent_v,
                                                         self.dense, self.dense_m, self.dense_v)])
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        check(kg_bind(self.h, C.byref(self.tables), C.c_void_p(self.stream.cuda_stream)), self.h)

    # -- calls -------------------------------------------------------------
    def init_params(self, seed):
        check(kg_init_params(self.h, seed), self.h)

    def set_apply(self, apply=True, keep_grads=False, stage_timing=False):
        check(kg_set_apply(self.h, int(apply) | (int(keep_grads) << 1) | (int(stage_timing) << 2)), self.h)

    @staticmethod
    def batch_struct(b, on_device=False) -> kg_batch:
        keep = [b["anchors"], b["relations"], b.get("answers"), b.get("negatives"), b.get("mask")]
        s = kg_batch(STRUCTS[b["structure"]], int(b["M"]), int(b.get("K", 0)),
                     *[_ptr(x) for x in keep], int(on_device))
        s._keep = keep
        return s

    @staticmethod
    def host_batch(b) -> dict:
        """Contiguous numpy arrays with the ABI dtypes."""
        return dict(structure=b["structure"], M=int(b["M"]), K=int(b["K"]),
                    anchors=np.ascontiguousarray(b["anchors"], np.int64),
                    relations=np.ascontiguousarray(b["relations"], np.int32),
                    answers=np.ascontiguousarray(b["answers"], np.int64),
                    negatives=np.ascontiguousarray(b["negatives"], np.int64),
                    mask=np.ascontiguousarray(b["mask"], np.uint32))

    def device_batch(self, b) -> dict:
        t = self.torch
        hb = self.host_batch(b)
        out = dict(structure=b["structure"], M=hb["M"], K=hb["K"])
        for k in ("anchors", "relations", "answers", "negatives", "mask"):
            a = hb[k]
            if a.dtype == np.uint32:
                a = a.view(np.int32)
            out[k] = t.from_numpy(a.copy()).to(self.dense.device)
        return out

    def step(self, b, lr, sync=True, on_device=False):
        bs = self.batch_struct(b, on_device)
        info = kg_step_info()
        st = kg_step(self.h, C.byref(bs), C.c_float(lr), C.byref(info) if sync else None)
        check(st, self.h)
        return info if sync else None

    def sync(self):
        info = kg_step_info()
        check(kg_sync(self.h, C.byref(info)), self.h)
        return info

    def result(self):
        """The oldest unread step's result (pipelined loops: issue step s + 1, then read step s)."""
        info = kg_step_info()
        check(kg_result(self.h, C.byref(info)), self.h)
        return info

    def score(self, b, cand):
        cand = np.ascontiguousarray(cand, np.int64)
        bs = self.batch_struct(dict(b, K=0, answers=None, negatives=None, mask=None))
        out = np.empty((int(b["M"]), len(cand)), np.float32)
        check(kg_score(self.h, C.byref(bs), cand.ctypes.data, len(cand), out.ctypes.data), self.h)
        return out

    def score_each(self, b, cand):
        """kg_score_each: cand [M][n_cand] per-query candidates -> distances [M][n_cand]."""
        cand = np.ascontiguousarray(cand, np.int64)
        assert cand.ndim == 2 and cand.shape[0] == int(b["M"])
        bs = self.batch_struct(dict(b, K=0, answers=None, negatives=None, mask=None))
        out = np.empty(cand.shape, np.float32)
        check(kg_score_each(self.h, C.byref(bs), cand.ctypes.data, cand.shape[1], out.ctypes.data), self.h)
        return out

    def eval(self, b, ans_off, ans_ids, negatives):
        """kg_eval: (ranks [n_ans] int32, metrics [M][4] = MRR, Hit@1, Hit@3, Hit@10)."""
        ans_off = np.ascontiguousarray(ans_off, np.int64)
        ans_ids = np.ascontiguousarray(ans_ids, np.int64)
        negatives = np.ascontiguousarray(negatives, np.int64)
        M = int(b["M"])
        n_neg = negatives.shape[1] if negatives.ndim == 2 else 0
        bs = self.batch_struct(dict(b, K=0, answers=None, negatives=None, mask=None))
        ranks = np.empty(int(ans_off[-1]), np.int32)
        metrics = np.empty((M, 4), np.float32)
        check(kg_eval(self.h, C.byref(bs), ans_off.ctypes.data, ans_ids.ctypes.data, n_neg,
                      negatives.ctypes.data if n_neg else None, ranks.ctypes.data, metrics.ctypes.data), self.h)
        return ranks, metrics

    def read_rows(self, ids, which=0):
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.empty((len(ids), self.cfg.dim), np.float32)
        check(kg_read_rows(self.h, which, ids.ctypes.data, len(ids), out.ctypes.data), self.h)
        return out

    def gather_rows(self, ids, which=0):
        """Collective (world > 1: every rank calls it): rows of any global ids, from their owners."""
        ids = np.ascontiguousarray(ids, np.int64)
        out = np.empty((len(ids), self.cfg.dim), np.float32)
        check(kg_gather_rows(self.h, which, ids.ctypes.data if len(ids) else None, len(ids),
                             out.ctypes.data if len(ids) else None), self.h)
        return out

    def write_rows(self, ids, rows, which=0):
        ids = np.ascontiguousarray(ids, np.int64)
        rows = np.ascontiguousarray(rows, np.float32)
        check(kg_write_rows(self.h, which, ids.ctypes.data, len(ids), rows.ctypes.data), self.h)

    def read_dense(self, which=0):
        out = np.empty(self.dense_size, np.float32)
        check(kg_read_dense(self.h, which, out.ctypes.data), self.h)
        return out

    def write_dense(self, x, which=0):
        x = np.ascontiguousarray(x, np.float32)
        assert x.size == self.dense_size
        check(kg_write_dense(self.h, which, x.ctypes.data), self.h)

    def last_grads(self, cap, M=None, K=None):
        uniq = np.empty(cap, np.int64)
        g = np.empty((cap, self.cfg.dim), np.float32)
        gd = np.empty(self.dense_size, np.float32)
        n = C.c_int32()
        dpos = np.empty(M, np.float32) if M else None
        dneg = np.empty((M, K), np.float32) if (M and K) else None
        check(kg_last_grads(self.h, uniq.ctypes.data, g.ctypes.data, gd.ctypes.data, cap, C.byref(n),
                            None if dpos is None else dpos.ctypes.data,
                            None if dneg is None else dneg.ctypes.data), self.h)
        U = n.value
        return dict(uniq=uniq[:U], grad_rows=g[:U], grad_dense=gd, d_pos=dpos, d_neg=dneg)

    # -- checkpoint / resume (the tables are this object's tensors; t is the library's) --------
    def get_step(self) -> int:
        t = C.c_int64()
        check(kg_get_step(self.h, C.byref(t)), self.h)
        return t.value

    def save(self, path):
        """theta_E shard, theta_D, their Adam moments and the Adam step counter, with torch.save."""
        torch = self.torch
        state = {k: getattr(self, k).detach().cpu() for k in ("ent", "ent_m", "ent_v", "dense", "dense_m", "dense_v")}
        state["t"] = self.get_step()
        state["dim"], state["rows"] = self.cfg.dim, self.rows
        torch.save(state, path)

    def load(self, path):
        torch = self.torch
        state = torch.load(path, weights_only=True)
        assert state["dim"] == self.cfg.dim and state["rows"] == self.rows, "checkpoint of another shape"
        torch.cuda.synchronize()
        for k in ("ent", "ent_m", "ent_v", "dense", "dense_m", "dense_v"):
            getattr(self, k).copy_(state[k])
        torch.cuda.synchronize()
        check(kg_set_step(self.h, int(state["t"])), self.h)

    def close(self):
        if self.h:
            kg_destroy(self.h)
            self.h = _H()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
