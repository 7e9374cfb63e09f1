"""Forward definitions of the query-embedding models, fp64 (TEST INFRASTRUCTURE ONLY).

Each function restates a row of PAPER.md Table 1 (multi-hop models)
or Table 2 (single-hop models) with the readings listed in
DESIGN.md §"Readings of the paper" (A-numbers).  Storage conventions (A1):

  * an entity row x has d floats for every model;
  * BetaE: e(x) = clamp(x + 1, 0.05, 1e9), alpha = e[:m], beta = e[m:], m = d/2 (A1, A8);
  * RotatE / ComplEx: complex vector of m = d/2 entries stored [re | im] (A1);
  * Q2B: a query is a box [center | offset] (2d floats); an entity is a point
    (offset 0) (A6, Table 1 "q in R^{2d}, v in R^d").

theta_D (relation tables + operator weights) is a flat array; `dense_views`
slices it by kggen.dense_layout.
"""
from __future__ import annotations

import torch

import kggen

F64 = torch.float64


def dense_views(cfg: kggen.ModelConfig, theta: torch.Tensor) -> dict:
    """name -> view of the flat theta_D tensor (layout of kggen.dense_layout)."""
    offs, total = kggen.dense_offsets(cfg)
    assert theta.numel() == total
    return {name: theta[o:o + int(torch.tensor(shape).prod())].view(*shape)
            for name, (o, shape) in offs.items()}


def _linear(x, W, b):
    """y = W x + b for row vectors x (W stored [out][in])."""
    return x @ W.T + b


# Test instrumentation (no arithmetic change): when TRACE is a list, every discrete decision
# the forward takes on a computed value -- a ReLU / clamp kink or an argmin between inputs --
# appends (margin, scale): the signed distance of the value from the kink and the magnitude
# scale of the sum that produced it (|W| |x| + |b|).  tests/test_fullsize_gpu.py uses it to
# build inputs whose decisions are well away from fp32 rounding (reading A28).
TRACE = None


def _trace(margin, scale):
    if TRACE is not None:
        TRACE.append((margin.detach(), scale.detach()))


def _relu_lin(x, W, b):
    """ReLU(W x + b), traced at its kink."""
    z = _linear(x, W, b)
    if TRACE is not None:
        _trace(z, x.abs() @ W.abs().T + b.abs())
    return torch.relu(z)


def _halves(x):
    m = x.shape[-1] // 2
    return x[..., :m], x[..., m:]


def _base(kind: str) -> str:
    """The -m multi-hop variants (App. B) project and score like their base model."""
    return kggen.M_VARIANTS.get(kind, kind)


def normalize(kind: str, q: torch.Tensor) -> torch.Tensor:
    """App. B: DistMult-m q / ||q||_2; ComplEx-m Re and Im parts each to the unit
    sphere; identity for every other kind (RotatE-m is not normalised, reading A27)."""
    if kind == "distmult-m":
        return q / torch.linalg.vector_norm(q, dim=-1, keepdim=True)
    if kind == "complex-m":
        re, im = _halves(q)
        return torch.cat([re / torch.linalg.vector_norm(re, dim=-1, keepdim=True),
                          im / torch.linalg.vector_norm(im, dim=-1, keepdim=True)], dim=-1)
    return q


# ---------------------------------------------------------------- embeddings
def embed_entity(kind: str, x: torch.Tensor) -> torch.Tensor:
    """Entity embedding Em(v) from a raw row (Table 1/2 'Embedding Space')."""
    if kind == "betae":
        # A8: Beta parameters must be positive; e(x) = clamp(x + 1, 0.05, 1e9)
        return torch.clamp(x + 1.0, 0.05, 1e9)
    return x


def anchor_query(kind: str, x: torch.Tensor) -> torch.Tensor:
    """Query embedding of an anchor node (a leaf of the computation plan)."""
    if kind == "q2b":
        # A6: an anchor is a point, i.e. a box with zero offset.
        return torch.cat([x, torch.zeros_like(x)], dim=-1)
    return embed_entity(kind, x)


# ---------------------------------------------------------------- projection
def project(kind: str, q: torch.Tensor, r: torch.Tensor, P: dict) -> torch.Tensor:
    """Relation projection P(q, r) (Table 1 'Relation Projection', App. B).

    q: [M, dq] query embeddings, r: int64 [M] relation ids.
    """
    if kind in kggen.M_VARIANTS:   # base projection, then the -m normalisation
        return normalize(kind, project(_base(kind), q, r, P))
    if kind in ("gqe", "transe"):
        return q + P["rel"][r]                                  # Em(q) + Em(r)
    if kind == "q2b":
        d = q.shape[-1] // 2
        c, o = q[..., :d], q[..., d:]
        # A6: center translates, offset grows by ReLU(offset row) (stays >= 0)
        return torch.cat([c + P["rel_center"][r], o + torch.relu(P["rel_offset"][r])], dim=-1)
    if kind == "betae":
        # Table 1 MLP(Em(q), Em(r)); A9: [e_q; y] -> H -> H -> d, ReLU, A8 clamp(+1)
        x = torch.cat([q, P["rel"][r]], dim=-1)
        h1 = _relu_lin(x, P["prj_W1"], P["prj_b1"])
        h2 = _relu_lin(h1, P["prj_W2"], P["prj_b2"])
        y = _linear(h2, P["prj_W0"], P["prj_b0"])
        if TRACE is not None:
            _trace(y + 1.0 - 0.05, h2.abs() @ P["prj_W0"].abs().T + P["prj_b0"].abs() + 1.0)
        return torch.clamp(y + 1.0, 0.05, 1e9)
    if kind == "rotate":
        # Table 2 h o r with |r_k| = 1; A3: r_k = exp(i theta_k)
        h_re, h_im = _halves(q)
        th = P["rel_phase"][r]
        c, s = torch.cos(th), torch.sin(th)
        return torch.cat([h_re * c - h_im * s, h_re * s + h_im * c], dim=-1)
    if kind == "distmult":
        return q * P["rel"][r]                                  # h o r (real)
    if kind == "complex":
        h_re, h_im = _halves(q)
        r_re, r_im = _halves(P["rel"][r])
        return torch.cat([h_re * r_re - h_im * r_im, h_re * r_im + h_im * r_re], dim=-1)
    raise ValueError(kind)


# -------------------------------------------------------------- intersection
def intersect(kind: str, qs: list, P: dict) -> torch.Tensor:
    """Intersection I({q_i}) (Table 1 'Intersection'; A4, A5)."""
    X = torch.stack(qs, dim=0)                                  # [n, M, dq]
    if kind in kggen.M_VARIANTS:
        # GQE's DeepSet on the d-float rows ([re | im] for the complex ones)
        h = _relu_lin(X, P["ds_W1"], P["ds_b1"]).mean(dim=0)
        return normalize(kind, _linear(h, P["ds_W2"], P["ds_b2"]))
    if kind == "gqe":
        # A4 DeepSet: W2 * mean_i ReLU(W1 q_i + b1) + b2
        h = _relu_lin(X, P["ds_W1"], P["ds_b1"]).mean(dim=0)
        return _linear(h, P["ds_W2"], P["ds_b2"])
    if kind == "q2b":
        d = X.shape[-1] // 2
        C, O = X[..., :d], X[..., d:]
        # A5 center: a_i = softmax_i(W2 ReLU(W1 c_i + b1) + b2); c = sum_i a_i * c_i
        logits = _linear(_relu_lin(C, P["att_W1"], P["att_b1"]), P["att_W2"], P["att_b2"])
        a = torch.softmax(logits, dim=0)
        c = (a * C).sum(dim=0)
        # Table 1: Off(q) = min({Off(q_i)}) * sigmoid(DeepSet({Off(q_i)}))  (A4 DeepSet)
        omin = O.min(dim=0).values                               # ties -> lowest index (A19)
        if TRACE is not None:
            for i in range(1, O.shape[0]):
                for j in range(i):   # exact ties are decided alike on both sides (same inputs)
                    gap = O[i] - O[j]
                    _trace(torch.where(gap == 0, torch.ones_like(gap), gap), O[i].abs() + O[j].abs())
        z = _linear(_relu_lin(O, P["off_W1"], P["off_b1"]).mean(dim=0),
                    P["off_W2"], P["off_b2"])
        return torch.cat([c, omin * torch.sigmoid(z)], dim=-1)
    if kind == "betae":
        # Table 1: [(sum w_i alpha_i, sum w_i beta_i)]; A5: w = softmax_i(U2 ReLU(U1 [a_i; b_i] + c1) + c2)
        logits = _linear(_relu_lin(X, P["att_U1"], P["att_c1"]), P["att_U2"], P["att_c2"])
        w = torch.softmax(logits, dim=0)                         # [n, M, m]
        A, B = _halves(X)
        return torch.cat([(w * A).sum(dim=0), (w * B).sum(dim=0)], dim=-1)
    raise ValueError(f"{kind} has no intersection operator in this build")


# ------------------------------------------------------------------ distance
def _ln_beta(a, b):
    return torch.lgamma(a) + torch.lgamma(b) - torch.lgamma(a + b)


def beta_kl(a1, b1, a2, b2):
    """KL(Beta(a1, b1) || Beta(a2, b2)), the closed form of the KL between Beta laws."""
    return (_ln_beta(a2, b2) - _ln_beta(a1, b1)
            + (a1 - a2) * torch.digamma(a1) + (b1 - b2) * torch.digamma(b1)
            + (a2 - a1 + b2 - b1) * torch.digamma(a1 + b1))


def distance(kind: str, q: torch.Tensor, v: torch.Tensor, box_alpha: float = 0.02) -> torch.Tensor:
    """Dist(q, Em(v)) for query embeddings q [..., dq] and RAW entity rows v [..., d]
    (broadcasting over leading dims).  Lower = closer (A13 for the semantic-matching kinds)."""
    kind = _base(kind)
    if kind in ("gqe", "transe"):
        # App. B P:L624 ||q - v||_2 ; Table 2 ||h + r - t|| (A2: L2)
        return torch.linalg.vector_norm(q - v, dim=-1)
    if kind == "q2b":
        d = v.shape[-1]
        c, o = q[..., :d], q[..., d:]
        delta = (v - c).abs()
        # A7: dist_out = sum ReLU(|v - c| - o); dist_in = sum min(|v - c|, o) (tie -> o, A19)
        dist_out = torch.relu(delta - o).sum(dim=-1)
        dist_in = torch.where(delta < o, delta, o).sum(dim=-1)
        return dist_out + box_alpha * dist_in
    if kind == "betae":
        # Table 1: KL(Beta(Em(v)); Beta(Em(q))), entity first (A10)
        a1, b1 = _halves(embed_entity(kind, v))
        a2, b2 = _halves(q)
        return beta_kl(a1, b1, a2, b2).sum(dim=-1)
    if kind == "rotate":
        # Table 2 ||h o r - t||, A3: sum of complex moduli
        z_re, z_im = _halves(q - v)
        return torch.linalg.vector_norm(torch.stack([z_re, z_im], dim=-1), dim=-1).sum(dim=-1)
    if kind == "distmult":
        return -(q * v).sum(dim=-1)                              # -<h o r, t>
    if kind == "complex":
        q_re, q_im = _halves(q)
        v_re, v_im = _halves(v)
        return -(q_re * v_re + q_im * v_im).sum(dim=-1)          # -Re<h o r, conj(t)>
    raise ValueError(kind)


# ------------------------------------------------------------------ negation
def negate(kind: str, q: torch.Tensor) -> torch.Tensor:
    """Negation N(q) = 1 / Em(q) on the Beta parameters (Table 1); BetaE only."""
    if kind != "betae":
        raise ValueError(f"{kind} has no negation operator (Table 1 'Negation' column is '-')")
    return 1.0 / q


# --------------------------------------------------------------- query DAGs
def query_disjuncts(structure: str, kind: str, anchors: list, rels: list, P: dict) -> list:
    """Evaluate the computation plan of a structure bottom-up (the
    negation structures 2in / 3in / inp / pin / pni of P:L775 use N(q) = 1/q, BetaE only).

    anchors: list (per anchor slot, execution order) of RAW rows [M, d];
    rels: list (per relation slot, execution order A21) of int64 [M].
    Returns the list of DNF disjunct query embeddings (Def. 1; unions
    are kept as separate disjuncts, 'DNF' columns of Table 8, A11).
    """
    A = [anchor_query(kind, x) for x in anchors]

    def p(q, s):
        return project(kind, q, rels[s], P)

    def i(*qs):
        return intersect(kind, list(qs), P)

    s = structure
    if s == "1p":
        return [p(A[0], 0)]
    if s == "2p":
        return [p(p(A[0], 0), 1)]
    if s == "3p":
        return [p(p(p(A[0], 0), 1), 2)]
    if s == "2i":
        return [i(p(A[0], 0), p(A[1], 1))]
    if s == "3i":
        return [i(p(A[0], 0), p(A[1], 1), p(A[2], 2))]
    if s == "ip":
        return [p(i(p(A[0], 0), p(A[1], 1)), 2)]
    if s == "pi":
        return [i(p(p(A[0], 0), 1), p(A[1], 2))]
    if s == "2u":
        return [p(A[0], 0), p(A[1], 1)]
    if s == "up":
        # (p (u (p a0) (p a1))) in DNF: the final relation r2 applies to both branches
        return [p(p(A[0], 0), 2), p(p(A[1], 1), 2)]

    def n(q):
        return negate(kind, q)

    # negation structures (BetaE): n marks the negated branch
    if s == "2in":
        return [i(p(A[0], 0), n(p(A[1], 1)))]
    if s == "3in":
        return [i(p(A[0], 0), p(A[1], 1), n(p(A[2], 2)))]
    if s == "inp":
        return [p(i(p(A[0], 0), n(p(A[1], 1))), 2)]
    if s == "pin":
        return [i(p(p(A[0], 0), 1), n(p(A[1], 2)))]
    if s == "pni":
        return [i(n(p(p(A[0], 0), 1)), p(A[1], 2))]
    raise ValueError(s)
