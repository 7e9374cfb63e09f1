"""One training step, written out plainly in fp64 (TEST INFRASTRUCTURE ONLY).

Follows the worker loop of PAPER.md §4.1 P:L303-309 (collect batch -> load
rows -> gradients, AllReduce of dL/dtheta_D, update theta_D -> update theta_E),
synchronously (reading A18), with

  * Eq. 1 loss over the shared-negative batch format of §4.3
    P:L389 (reading A12: l_i = softplus(D+_i - gamma) + (1/n_i) sum_j mask_ij
    softplus(gamma - D_ij), n_i = popcount of mask row i; batch loss = mean);
  * the duplicate-row merge of P:L343 ('scatter ... into a single continuous
    memory'), i.e. one gradient row per distinct id;
  * Adam (Kingma-Ba) applied lazily to the touched rows of theta_E
    (A16) and to every element of theta_D (A17),
    textbook bias correction (A15).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import kggen
from .model import F64, dense_views, distance, query_disjuncts


# ---------------------------------------------------------------- utilities
def softplus(z: torch.Tensor) -> torch.Tensor:
    """softplus(z) = log(1 + e^z) = -log sigmoid(-z), evaluated without overflow.

    Two smooth branches (each differentiated by autograd away from its clamp), so
    the derivative at z = 0 is sigmoid(0) = 1/2 exactly (pinned by the P3 worked
    example, where gamma - D_j = 0).
    """
    pos = torch.clamp(z, min=0.0)
    neg = torch.clamp(z, max=0.0)
    return torch.where(z > 0, pos + torch.log1p(torch.exp(-pos)), torch.log1p(torch.exp(neg)))


def dedup(ids: np.ndarray):
    """P:L343 merge: distinct ids ascending and the inverse map (plain definition)."""
    ids = np.asarray(ids, dtype=np.int64).reshape(-1)
    uniq = np.array(sorted(set(ids.tolist())), dtype=np.int64)
    inv = np.searchsorted(uniq, ids).astype(np.int64)
    return uniq, inv


def adam(p, m, v, g, lr, t, beta1, beta2, eps):
    """Adam (Kingma & Ba), textbook form with bias correction (reading A15), fp64."""
    p = np.asarray(p, dtype=np.float64)
    m = beta1 * np.asarray(m, dtype=np.float64) + (1.0 - beta1) * g
    v = beta2 * np.asarray(v, dtype=np.float64) + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** t)
    v_hat = v / (1.0 - beta2 ** t)
    p = p - lr * m_hat / (np.sqrt(v_hat) + eps)
    return p, m, v


class SparseTable:
    """theta_E and its Adam moments as {id: row} over the pure-function init (A23).

    Rows never written read as their init value (moments 0), so a Freebase-shaped
    step needs only the touched rows.  Values are stored as float32 (A24).
    """

    def __init__(self, cfg: kggen.ModelConfig, seed: int, dense: np.ndarray = None):
        self.cfg, self.seed = cfg, seed
        self.rows = {}
        self.dense = (kggen.init_dense(cfg, seed) if dense is None else np.asarray(dense, np.float32)).copy()
        self.dense_m = np.zeros_like(self.dense)
        self.dense_v = np.zeros_like(self.dense)
        self.t = 0

    def get(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        d = self.cfg.dim
        p = kggen.init_entity_rows(self.cfg, self.seed, ids)
        m = np.zeros((len(ids), d), np.float32)
        v = np.zeros((len(ids), d), np.float32)
        for k, i in enumerate(ids.tolist()):
            if i in self.rows:
                p[k], m[k], v[k] = self.rows[i]
        return p, m, v

    def set(self, ids, p, m, v):
        for k, i in enumerate(np.asarray(ids, dtype=np.int64).tolist()):
            self.rows[i] = (np.float32(p[k]), np.float32(m[k]), np.float32(v[k]))


@dataclass
class StepResult:
    loss: float
    uniq: np.ndarray            # touched ids, ascending (A16)
    grad_rows: np.ndarray       # [U, d] merged dL/dtheta_E rows (fp64)
    grad_dense: np.ndarray      # [|theta_D|] dL/dtheta_D (fp64)
    d_pos: list                 # per rank: [M] D+ (DNF min)
    d_neg: list                 # per rank: [M, K] D (DNF min, unmasked)
    rows_new: np.ndarray = None  # [U, d] fp64 p, m, v after Adam
    m_new: np.ndarray = None
    v_new: np.ndarray = None
    dense_new: np.ndarray = None
    dense_m_new: np.ndarray = None
    dense_v_new: np.ndarray = None


def _batch_ids(b):
    return np.concatenate([np.asarray(b["anchors"], np.int64).reshape(-1),
                           np.asarray(b["answers"], np.int64).reshape(-1),
                           np.asarray(b["negatives"], np.int64).reshape(-1)])


def query_loss_terms(cfg, structure, P, X, slot_inv, rels, mask_bits, lo, hi, M, G):
    """Per-query Eq. 1 terms for queries [lo, hi) of one rank's batch.

    X: [U, d] leaf of distinct raw rows; slot_inv: dict of inverse-map index
    arrays for 'anchors' [M, na], 'answers' [M], 'negatives' [K].
    Returns (sum_i l_i / (M G), D+ [hi-lo], D [hi-lo, K]).
    """
    na = kggen.N_ANCHORS[structure]
    anchors = [X[torch.as_tensor(slot_inv["anchors"][lo:hi, a])] for a in range(na)]
    rel = [torch.as_tensor(rels[lo:hi, s].astype(np.int64)) for s in range(rels.shape[1])]
    qs = query_disjuncts(structure, cfg.kind, anchors, rel, P)
    v_pos = X[torch.as_tensor(slot_inv["answers"][lo:hi])]                  # [m, d]
    v_neg = X[torch.as_tensor(slot_inv["negatives"])]                       # [K, d]
    # DNF union (A11): distance to a union = min over its disjuncts, per candidate
    d_pos = torch.stack([distance(cfg.kind, q, v_pos, cfg.box_alpha) for q in qs]).min(dim=0).values
    d_neg = torch.stack([distance(cfg.kind, q[:, None, :], v_neg[None, :, :], cfg.box_alpha)
                         for q in qs]).min(dim=0).values                     # [m, K]
    mask = torch.as_tensor(mask_bits[lo:hi]).to(F64)
    n_i = mask.sum(dim=1)
    neg_term = (mask * softplus(cfg.gamma - d_neg)).sum(dim=1) / torch.clamp(n_i, min=1.0)
    loss_i = softplus(d_pos - cfg.gamma) + neg_term                          # Eq. 1 with |A| = 1
    return loss_i.sum() / (M * G), d_pos.detach(), d_neg.detach()


def oracle_step(cfg: kggen.ModelConfig, table: SparseTable, batches: list, lr: float,
                apply: bool = True, pair_budget: int = 2_000_000) -> StepResult:
    """One synchronous step over G = len(batches) workers (A18), optional update.

    Global loss L = (1/G) sum_w (1/M) sum_i l_i; dL/dtheta summed over workers;
    one Adam update of every touched row and of theta_D; t += 1.
    """
    G = len(batches)
    structure = batches[0]["structure"]
    assert all(b["structure"] == structure for b in batches), "one structure per step (P:L398)"
    ids_all = np.concatenate([_batch_ids(b) for b in batches])
    uniq, inv_all = dedup(ids_all)
    p0, m0, v0 = table.get(uniq)
    X = torch.tensor(p0, dtype=F64, requires_grad=True)
    theta = torch.tensor(table.dense, dtype=F64, requires_grad=True)
    P = dense_views(cfg, theta)

    total = 0.0
    d_pos_all, d_neg_all = [], []
    off = 0
    for b in batches:
        M, K = len(b["answers"]), int(b["K"])
        na = kggen.N_ANCHORS[structure]
        n_ids = M * na + M + K
        inv = inv_all[off:off + n_ids]
        off += n_ids
        slot_inv = {"anchors": inv[:M * na].reshape(M, na),
                    "answers": inv[M * na:M * na + M],
                    "negatives": inv[M * na + M:]}
        bits = kggen.unpack_mask(np.asarray(b["mask"]), K)
        rels = np.asarray(b["relations"])
        chunk = max(1, pair_budget // max(1, K * cfg.dim))
        dp, dn = [], []
        for lo in range(0, M, chunk):
            hi = min(M, lo + chunk)
            lsum, d_pos, d_neg = query_loss_terms(cfg, structure, P, X, slot_inv, rels, bits,
                                                  lo, hi, M, G)
            lsum.backward()       # gradient of a sum = sum of per-chunk gradients
            total += float(lsum.detach())
            dp.append(d_pos.numpy())
            dn.append(d_neg.numpy())
        d_pos_all.append(np.concatenate(dp))
        d_neg_all.append(np.concatenate(dn) if dn else np.zeros((0, K)))

    gE = X.grad.numpy().copy() if X.grad is not None else np.zeros_like(p0, np.float64)
    gD = theta.grad.numpy().copy() if theta.grad is not None else np.zeros(table.dense.shape)
    res = StepResult(loss=total, uniq=uniq, grad_rows=gE, grad_dense=gD,
                     d_pos=d_pos_all, d_neg=d_neg_all)
    if apply:
        t = table.t + 1
        res.rows_new, res.m_new, res.v_new = adam(p0, m0, v0, gE, lr, t, cfg.beta1, cfg.beta2, cfg.eps)
        res.dense_new, res.dense_m_new, res.dense_v_new = adam(
            table.dense, table.dense_m, table.dense_v, gD, lr, t, cfg.beta1, cfg.beta2, cfg.eps)
        table.t = t
        table.set(uniq, res.rows_new, res.m_new, res.v_new)
        table.dense = res.dense_new.astype(np.float32)
        table.dense_m = res.dense_m_new.astype(np.float32)
        table.dense_v = res.dense_v_new.astype(np.float32)
    return res


def oracle_score(cfg: kggen.ModelConfig, table: SparseTable, batch: dict, cand) -> np.ndarray:
    """Dist(f(q_i), f(v_c)) for every query i and shared candidate c, DNF min."""
    structure = batch["structure"]
    cand = np.asarray(cand, np.int64)
    M = len(batch["answers"]) if "answers" in batch else np.asarray(batch["anchors"]).shape[0]
    with torch.no_grad():
        theta = torch.tensor(table.dense, dtype=F64)
        P = dense_views(cfg, theta)
        anchors_ids = np.asarray(batch["anchors"], np.int64)
        anchors = [torch.tensor(table.get(anchors_ids[:, a])[0], dtype=F64)
                   for a in range(anchors_ids.shape[1])]
        rels = np.asarray(batch["relations"])
        rel = [torch.as_tensor(rels[:, s].astype(np.int64)) for s in range(rels.shape[1])]
        qs = query_disjuncts(structure, cfg.kind, anchors, rel, P)
        V = torch.tensor(table.get(cand)[0], dtype=F64)
        out = np.empty((M, len(cand)))
        chunk = max(1, 2_000_000 // max(1, len(cand) * cfg.dim))
        for lo in range(0, M, chunk):
            hi = min(M, lo + chunk)
            D = torch.stack([distance(cfg.kind, q[lo:hi, None, :], V[None], cfg.box_alpha)
                             for q in qs]).min(dim=0).values
            out[lo:hi] = D.numpy()
    return out


def oracle_score_each(cfg: kggen.ModelConfig, table: SparseTable, batch: dict, cand) -> np.ndarray:
    """Per-query candidates (SURVEY §8(b) kg_score with shared = 0): D[i, c] = Dist(f(q_i),
    f(v_{cand[i, c]})) with the DNF min over q_i's disjuncts (A11); cand [M][n_cand].
    Written out query by query (a plain loop over i), no tiling."""
    structure = batch["structure"]
    cand = np.asarray(cand, np.int64)
    M, n = cand.shape
    with torch.no_grad():
        theta = torch.tensor(table.dense, dtype=F64)
        P = dense_views(cfg, theta)
        anchors_ids = np.asarray(batch["anchors"], np.int64)
        anchors = [torch.tensor(table.get(anchors_ids[:, a])[0], dtype=F64)
                   for a in range(anchors_ids.shape[1])]
        rels = np.asarray(batch["relations"])
        rel = [torch.as_tensor(rels[:, s].astype(np.int64)) for s in range(rels.shape[1])]
        qs = query_disjuncts(structure, cfg.kind, anchors, rel, P)
        out = np.empty((M, n))
        for i in range(M):
            V = torch.tensor(table.get(cand[i])[0], dtype=F64)          # this query's candidates
            D = torch.stack([distance(cfg.kind, q[i:i + 1], V, cfg.box_alpha) for q in qs]).min(dim=0).values
            out[i] = D.numpy()
    return out

