"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu).

One kg_step per case at the workload's own M, K, d, |V| (the C5 per-GPU shard of
10,756,769 rows), |R| and MLP width, checked against the fp64 oracle on the same seeded
batch: the loss, every D+ and D_ij, the touched-row set (bit-exact), every merged row
gradient, the whole dL/dtheta_D, and the updated rows / theta_D (tolerances and the
Adam-first-step exclusion as in test_parity_gpu.py).  The oracle runs the full step
(C5 Q2B: ~20-40 s of CPU on the box), so every output is compared, not a sample.

Discrete decisions (reading A28).  Q2B's distance has two kinks per (query,
candidate, unit) term -- |t| = o (in-box / out-box) and t = 0 (the sign of t = v - c)
-- and the GPU takes them in fp32, the oracle in fp64.  At full size (10^8 terms) a few
terms lie within fp32 resolution of a kink, and a flipped decision moves one gradient
contribution by a jump of at most 2 |dL/dD| (dL/dD <= 1/M for a positive term,
<= 1/(M n_i) for a pool term, Eq. 1).  So for Q2B the test counts, in fp64 from the
oracle's own forward values, the terms within delta = 1e-5 (|c| + |o| + |v|) of a kink
(fp32 carries ~6e-8 relative error per op, a few ops deep), and lets at most 8 x that
many gradient elements per tensor exceed the rtol bound, each by at most twice the
largest jump among those terms.  Every other element keeps the plain 1e-5 bound; the
other models have no kinks inside their domains and get no allowance.  The DNF union
(2u / up) decides an argmin between disjuncts per (query, candidate); union batches are
made well-conditioned instead: pairs whose two disjunct distances are within 1e-5
relative are masked out of the pool (they carry no loss term), and a seed whose
positives have such a tie is skipped (an fp32 torch re-run of the oracle flips those
decisions too).  The same holds for every other discrete decision the forward takes on
a computed value -- the ReLUs of the BetaE projection MLP, of the attention / DeepSet
MLPs, the clamp of the BetaE projection output, the min over Q2B offsets: a flipped
ReLU moves a whole row of dW by a few percent.  So the batch is conditioned: queries whose
fp64 pre-activations or argmin gaps sit within 2e-6 of the magnitude of the sum that
produced them are re-drawn (same recipe, same pool), see well_conditioned_batch.
"""
import contextlib

import numpy as np
import pytest
import torch

import kggen
import oracle

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def assert_close(x, ref, rtol=RTOL, what="", mask=None):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    assert x.shape == ref.shape, (what, x.shape, ref.shape)
    err = np.abs(x - ref)
    tol = rtol * np.abs(ref) + rtol * np.abs(ref).max()
    bad = err > tol
    if mask is not None:
        bad &= mask
    if bad.any():
        k = np.unravel_index(np.argmax(np.where(bad, err / np.maximum(tol, 1e-300), 0)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()}/{bad.size} out of tolerance; worst at {k}: "
                             f"got {x[k]!r} ref {ref[k]!r}")


def q2b_flip_allowance(cfg, table, b, M, K, rel=1e-6):
    """Per-element allowance for Q2B's kinks, from the oracle itself (reading A28).

    A term (query i, candidate j, unit k) within rel * (|c| + |o| + |v|) of a kink -- |t| = o
    or t = 0, t = v - c -- may be decided the other way in fp32 (rel = 1e-6, ~16 ulp: the
    GPU's query boxes carry the rounding of a few fp32 ops and of the intersection MLPs).  A flip changes dD/dv, dD/dc
    and dD/do of that term by at most 1 (W in {0, alpha, 1}, dD/do = alpha - W), i.e. the
    adjoints of v_jk, c_ik and o_ik by at most |dL/dD_ij| (Eq. 1: sigma(gamma - D)/(M n_i) for
    a pool term, sigma(D+ - gamma)/M for the positive).  The candidate row's element (j, k)
    gets that bound directly; the query side is propagated exactly through the query's DAG
    with one vector-Jacobian product per flagged (i, k): allowance += w_ik |dc_ik/dtheta| +
    w_ik |do_ik/dtheta| on the anchor rows, relation rows and operator weights of query i.
    Every element no flagged term reaches gets no allowance (the plain 1e-5 bar).
    Returns (allow_rows [len(uniq), d] aligned with the oracle's uniq, allow_dense, n_terms)."""
    import torch
    import oracle.model as OM
    d = cfg.dim
    na = kggen.N_ANCHORS[b["structure"]]
    ids = np.concatenate([b["anchors"].reshape(-1), b["answers"], b["negatives"]])
    uniq, inv = oracle.dedup(ids)
    X = torch.tensor(table.get(uniq)[0], dtype=torch.float64)
    theta = torch.tensor(table.dense, dtype=torch.float64)
    P = OM.dense_views(cfg, theta)
    ia = inv[:M * na].reshape(M, na)
    rels = [torch.as_tensor(b["relations"][:, s].astype(np.int64)) for s in range(b["relations"].shape[1])]
    with torch.no_grad():
        qs = OM.query_disjuncts(b["structure"], cfg.kind, [X[torch.as_tensor(ia[:, a])] for a in range(na)], rels, P)
    dpos, dneg, _ = oracle_forward(cfg, table, b, M, K)
    bits = kggen.unpack_mask(b["mask"], K)
    n_i = bits.sum(axis=1).astype(np.float64)
    g = cfg.gamma
    sig = lambda z: 1.0 / (1.0 + np.exp(-z))  # noqa: E731
    c_pos = sig(dpos.min(axis=0) - g) / M                                       # [M]
    c_neg = np.where(bits, sig(g - dneg.min(axis=0)) / (M * np.maximum(n_i, 1))[:, None], 0.0)   # [M, K]
    arg_pos, arg_neg = dpos.argmin(axis=0), dneg.argmin(axis=0)
    vpos = X[torch.as_tensor(inv[M * na:M * na + M])]
    vneg = X[torch.as_tensor(inv[M * na + M:])]
    allow_rows = np.zeros((len(uniq), d))
    w = np.zeros((len(qs), M, d))                  # query-side weight per (disjunct, i, k)
    n_terms = 0
    pos_u, neg_u = inv[M * na:M * na + M], inv[M * na + M:]
    for t_, q in enumerate(qs):
        c, o = q[:, :d], q[:, d:]
        tt = vpos - c
        near = (((tt.abs() - o).abs() <= rel * (c.abs() + o.abs() + vpos.abs())) | (tt.abs() <= rel * (c.abs() + vpos.abs())))
        near = near.numpy() & (arg_pos == t_)[:, None]
        ii, kk = np.nonzero(near)
        n_terms += len(ii)
        np.add.at(allow_rows, (pos_u[ii], kk), c_pos[ii])
        np.add.at(w[t_], (ii, kk), c_pos[ii])
        for lo in range(0, M, 16):
            cc, oo = c[lo:lo + 16, None, :], o[lo:lo + 16, None, :]
            tt = vneg[None] - cc
            sc = rel * (cc.abs() + vneg[None].abs())
            near = ((tt.abs() - oo).abs() <= sc + rel * oo.abs()) | (tt.abs() <= sc)
            near = near.numpy() & ((arg_neg[lo:lo + 16] == t_) & bits[lo:lo + 16])[:, :, None]
            ii, jj, kk = np.nonzero(near)
            if len(ii):
                n_terms += len(ii)
                cw = c_neg[lo + ii, jj]
                np.add.at(allow_rows, (neg_u[jj], kk), cw)
                np.add.at(w[t_], (lo + ii, kk), cw)
    # the query side, through each flagged query's DAG (exact vector-Jacobian products)
    offs, total = kggen.dense_offsets(cfg)
    allow_dense = np.zeros(total)
    rel_names = [n for n in offs if n.startswith("rel")]
    wnames = [n for n in offs if not n.startswith("rel")]
    for t_ in range(len(qs)):
        for i in np.nonzero(w[t_].any(axis=1))[0]:
            rid = b["relations"][i].astype(np.int64)
            ur, rinv = np.unique(rid, return_inverse=True)
            leaves_a = [X[ia[i, a]].clone().view(1, d).requires_grad_(True) for a in range(na)]
            Pi = {n: P[n].detach().clone().requires_grad_(True) for n in wnames}
            leaves_r = {n: P[n][torch.as_tensor(ur)].detach().clone().requires_grad_(True) for n in rel_names}
            Pi.update(leaves_r)
            rels_i = [torch.as_tensor([int(rinv[s])]) for s in range(len(rid))]
            q = OM.query_disjuncts(b["structure"], cfg.kind, leaves_a, rels_i, Pi)[t_]
            leaves = leaves_a + [leaves_r[n] for n in rel_names] + [Pi[n] for n in wnames]
            for k in np.nonzero(w[t_, i])[0]:
                for col in (k, d + k):
                    gr = torch.autograd.grad(q[0, col], leaves, retain_graph=True, allow_unused=True)
                    for a in range(na):
                        if gr[a] is not None:
                            allow_rows[ia[i, a]] += w[t_, i, k] * gr[a].abs().numpy()[0]
                    for n, gg in zip(rel_names, gr[na:na + len(rel_names)]):
                        if gg is not None:
                            o0, shape = offs[n]
                            for r_, row in enumerate(ur):
                                allow_dense[o0 + row * shape[1]:o0 + (row + 1) * shape[1]] += \
                                    w[t_, i, k] * gg[r_].abs().numpy()
                    for n, gg in zip(wnames, gr[na + len(rel_names):]):
                        if gg is not None:
                            o0, shape = offs[n]
                            allow_dense[o0:o0 + gg.numel()] += w[t_, i, k] * gg.abs().reshape(-1).numpy()
    return allow_rows, allow_dense, n_terms


@contextlib.contextmanager
def _decision_hooks(rec):
    """Test-side hooks on the oracle's forward (no arithmetic change): every traced decision --
    a ReLU pre-activation, the BetaE projection clamp, a Q2B offset-min gap -- is recorded in
    call order as [margin, scale, post, kind] with the margin NOT detached and, for ReLU / clamp,
    the tensor the decision produced (post), so a per-query re-run can differentiate both."""
    import oracle.model as OM
    saved = (OM._trace, OM._relu_lin, OM.project, OM.TRACE)

    def tr(margin, scale):
        rec.append([margin, scale, None, "gap"])

    def rl(x, W, b_):
        z = OM._linear(x, W, b_)
        rec.append([z, x.abs() @ W.abs().T + b_.abs(), None, "relu"])
        out = torch.relu(z)
        if out.requires_grad:
            out.retain_grad()
        rec[-1][2] = out
        return out

    def pj(kind, q, r, P):
        out = saved[2](kind, q, r, P)
        if kind == "betae":              # project's last record is its clamp's margin
            rec[-1][3] = "clamp"
            if out.requires_grad:
                out.retain_grad()
            rec[-1][2] = out
        return out

    OM._trace, OM._relu_lin, OM.project, OM.TRACE = tr, rl, pj, []
    try:
        yield
    finally:
        OM._trace, OM._relu_lin, OM.project, OM.TRACE = saved


def traced_flip_allowance(cfg, table, b, M, K, rel=2e-6):
    """Per-element allowance for the forward's traced decisions taken on computed values (DESIGN.md
    reading A28): a ReLU pre-activation or the BetaE projection clamp within rel x the magnitude
    of the sum that produced it may fall the other way in fp32.  The value it produces moves by
    at most that margin (continuous), but the gradient through it switches between passing and
    blocking dL/d(post): the adjoint jump is |dL_i/d post| of the query's own loss term, and its
    effect on every parameter is |dL_i/d post| x |d margin / d theta|, one vector-Jacobian product
    per flagged (query, decision, unit) on the query's own DAG.  Q2B offset-min near-ties are not
    covered here (their queries are re-drawn).  Returns (allow_rows [len(uniq), d], allow_dense,
    number of flagged decisions)."""
    import oracle.model as OM
    d = cfg.dim
    na = kggen.N_ANCHORS[b["structure"]]
    ids = np.concatenate([b["anchors"].reshape(-1), b["answers"], b["negatives"]])
    uniq, inv = oracle.dedup(ids)
    X = torch.tensor(table.get(uniq)[0], dtype=torch.float64)
    theta = torch.tensor(table.dense, dtype=torch.float64)
    P = OM.dense_views(cfg, theta)
    ia = inv[:M * na].reshape(M, na)
    rels = [torch.as_tensor(b["relations"][:, s].astype(np.int64)) for s in range(b["relations"].shape[1])]
    rec = []
    with torch.no_grad(), _decision_hooks(rec):
        OM.query_disjuncts(b["structure"], cfg.kind, [X[torch.as_tensor(ia[:, a])] for a in range(na)], rels, P)
    flagged = {}   # query -> [(record index, index into the query's own tensor)]
    for k, (margin, scale, _, kind) in enumerate(rec):
        if kind == "gap":
            continue
        near = (margin.abs() <= rel * scale).numpy()
        for idx in zip(*np.nonzero(near)):
            if near.ndim == 2:          # [M, units]
                i, qidx = int(idx[0]), (0, int(idx[1]))
            else:                       # [n, M, units] (intersection inputs stacked)
                i, qidx = int(idx[1]), (int(idx[0]), 0, int(idx[2]))
            flagged.setdefault(i, []).append((k, qidx))
    offs, total = kggen.dense_offsets(cfg)
    allow_rows, allow_dense = np.zeros((len(uniq), d)), np.zeros(total)
    rel_names = [n for n in offs if n.startswith("rel")]
    wnames = [n for n in offs if not n.startswith("rel")]
    bits = kggen.unpack_mask(b["mask"], K)
    vpos_all = X[torch.as_tensor(inv[M * na:M * na + M])]
    vneg = X[torch.as_tensor(inv[M * na + M:])]
    g = cfg.gamma
    sp = lambda z: torch.nn.functional.softplus(z)  # noqa: E731
    n_flag = 0
    for i, items in flagged.items():
        rid = b["relations"][i].astype(np.int64)
        ur, rinv = np.unique(rid, return_inverse=True)
        leaves_a = [X[ia[i, a]].clone().view(1, d).requires_grad_(True) for a in range(na)]
        Pi = {n: P[n].detach().clone().requires_grad_(True) for n in wnames}
        leaves_r = {n: P[n][torch.as_tensor(ur)].detach().clone().requires_grad_(True) for n in rel_names}
        Pi.update(leaves_r)
        rels_i = [torch.as_tensor([int(rinv[s])]) for s in range(len(rid))]
        rq = []
        with _decision_hooks(rq):
            qs = OM.query_disjuncts(b["structure"], cfg.kind, leaves_a, rels_i, Pi)
        dp = torch.stack([OM.distance(cfg.kind, q, vpos_all[i:i + 1], cfg.box_alpha) for q in qs]).min(dim=0).values
        dn = torch.stack([OM.distance(cfg.kind, q[:, None, :], vneg[None], cfg.box_alpha) for q in qs]).min(dim=0).values
        mb = torch.as_tensor(bits[i], dtype=torch.float64)
        n_i = float(bits[i].sum())
        li = sp(dp - g).sum() + ((mb * sp(g - dn[0])).sum() / n_i if n_i > 0 else 0.0)
        li = li / M
        li.backward(retain_graph=True)
        leaves = leaves_a + [leaves_r[n] for n in rel_names] + [Pi[n] for n in wnames]
        for k, qidx in items:
            margin, _, post, _ = rq[k]
            if post is None or post.grad is None:
                continue
            jump = float(post.grad[qidx].abs())
            if jump == 0.0:
                continue
            n_flag += 1
            gr = torch.autograd.grad(margin[qidx], leaves, retain_graph=True, allow_unused=True)
            for a in range(na):
                if gr[a] is not None:
                    allow_rows[ia[i, a]] += jump * gr[a].abs().numpy()[0]
            for n, gg in zip(rel_names, gr[na:na + len(rel_names)]):
                if gg is not None:
                    o0, shape = offs[n]
                    for r_, row in enumerate(ur):
                        allow_dense[o0 + row * shape[1]:o0 + (row + 1) * shape[1]] += jump * gg[r_].abs().numpy()
            for n, gg in zip(wnames, gr[na + len(rel_names):]):
                if gg is not None:
                    o0, shape = offs[n]
                    allow_dense[o0:o0 + gg.numel()] += jump * gg.abs().reshape(-1).numpy()
    return allow_rows, allow_dense, n_flag


def oracle_forward(cfg, table, b, M, K, trace=False):
    """Oracle (fp64) forward of a batch: per-disjunct D+ [n, M], D [n, M, K], and the trace of
    the discrete decisions taken on computed values (oracle.model.TRACE) if asked."""
    import torch
    import oracle.model as OM
    na = kggen.N_ANCHORS[b["structure"]]
    ids = np.concatenate([b["anchors"].reshape(-1), b["answers"], b["negatives"]])
    uniq, inv = oracle.dedup(ids)
    X = torch.tensor(table.get(uniq)[0], dtype=torch.float64)
    P = OM.dense_views(cfg, torch.tensor(table.dense, dtype=torch.float64))
    ia = inv[:M * na].reshape(M, na)
    rels = [torch.as_tensor(b["relations"][:, s].astype(np.int64)) for s in range(b["relations"].shape[1])]
    OM.TRACE = [] if trace else None
    try:
        with torch.no_grad():
            qs = OM.query_disjuncts(b["structure"], cfg.kind, [X[torch.as_tensor(ia[:, a])] for a in range(na)],
                                    rels, P)
    finally:
        tr, OM.TRACE = OM.TRACE, None
    with torch.no_grad():
        vpos = X[torch.as_tensor(inv[M * na:M * na + M])]
        vneg = X[torch.as_tensor(inv[M * na + M:])]
        dpos = torch.stack([OM.distance(cfg.kind, q, vpos, cfg.box_alpha) for q in qs]).numpy()
        dneg = torch.stack([torch.cat([OM.distance(cfg.kind, q[lo:lo + 64, None, :], vneg[None, :, :], cfg.box_alpha)
                                       for lo in range(0, M, 64)]) for q in qs]).numpy()
    return dpos, dneg, tr


def _near(x, y):
    # exact ties are decided identically on both sides (same code on equal inputs -> the lowest
    # disjunct, A11); only near ties can flip between fp32 and fp64
    return (x != y) & (np.abs(x - y) <= 1e-5 * (np.abs(x) + np.abs(y)))


def _decision_kinds(cfg, table, b, M):
    """The kind ("relu" / "clamp" / "gap") of every traced decision of the batch, in call order."""
    import oracle.model as OM
    na = kggen.N_ANCHORS[b["structure"]]
    ids = np.concatenate([b["anchors"].reshape(-1), b["answers"], b["negatives"]])
    uniq, inv = oracle.dedup(ids)
    X = torch.tensor(table.get(uniq)[0], dtype=torch.float64)
    P = OM.dense_views(cfg, torch.tensor(table.dense, dtype=torch.float64))
    ia = inv[:M * na].reshape(M, na)
    rels = [torch.as_tensor(b["relations"][:, s].astype(np.int64)) for s in range(b["relations"].shape[1])]
    rec = []
    with torch.no_grad(), _decision_hooks(rec):
        OM.query_disjuncts(b["structure"], cfg.kind, [X[torch.as_tensor(ia[:, a])] for a in range(na)], rels, P)
    return [r[3] for r in rec]


def well_conditioned_batch(cfg, table, structure, M, K, seed):
    """A batch whose argmin decisions are well away from fp32 rounding (reading A28).

    Queries with a Q2B offset-min gap within 2e-6 of the magnitude of the values compared, or
    with a near-tie between the DNF disjuncts of their positive, are re-drawn from another batch
    of the same recipe (same pool); pool entries whose DNF disjunct distances nearly tie for a
    query are masked out for it (no loss term).  ReLU / clamp decisions are not re-drawn: the
    step is checked against their exact flip allowance (traced_flip_allowance).
    Returns (batch, number of re-drawn queries, number of masked pairs)."""
    b = {k: (v.copy() if isinstance(v, np.ndarray) else v)
         for k, v in kggen.make_batch(cfg, structure, M, K, seed=seed, step=0).items()}
    redrawn = 0
    for it in range(30):
        dpos, dneg, tr = oracle_forward(cfg, table, b, M, K, trace=True)
        kinds = _decision_kinds(cfg, table, b, M)
        assert len(kinds) == len(tr)
        bad = np.zeros(M, bool)
        for (margin, scale), kind in zip(tr, kinds):
            if kind != "gap":   # ReLU / clamp decisions: covered by traced_flip_allowance instead
                continue
            near = (margin.abs() <= 2e-6 * scale).numpy()
            bad |= near.reshape(-1, M, near.shape[-1]).any(axis=(0, 2)) if near.ndim >= 2 else near
        if len(dpos) == 2:
            bad |= _near(dpos[0], dpos[1])
        if not bad.any():
            break
        alt = kggen.make_batch(cfg, structure, M, K, seed=seed, step=1000 + it)
        idx = np.nonzero(bad)[0]
        redrawn += len(idx)
        for k in ("anchors", "relations", "answers"):
            b[k][idx] = alt[k][idx]
        bits = kggen.unpack_mask(b["mask"], K)
        bits[idx] &= b["negatives"][None, :] != b["answers"][idx, None]    # A20
        b["mask"] = kggen.pack_mask(bits)
    else:
        raise AssertionError("could not condition the batch")
    masked = 0
    if len(dneg) == 2:
        tie = _near(dneg[0], dneg[1])
        bits = kggen.unpack_mask(b["mask"], K)
        masked = int((bits & tie).sum())
        b["mask"] = kggen.pack_mask(bits & ~tie)
    return b, redrawn, masked


def assert_close_allow(x, ref, what, allow):
    """|x - ref| <= the plain bound + allow (elementwise; allow = 0 where no flagged term reaches)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    assert x.shape == ref.shape, (what, x.shape, ref.shape)
    err = np.abs(x - ref)
    tol = RTOL * np.abs(ref) + RTOL * np.abs(ref).max()
    bad = err > tol + allow
    if bad.any():
        k = np.unravel_index(np.argmax(np.where(bad, err - tol - allow, -np.inf)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()}/{bad.size} out of tolerance; worst at {k}: got {x[k]!r} ref "
                             f"{ref[k]!r}, allowance {allow[k]!r}")
    return int(((err > tol) & (allow > 0)).sum()), int((allow > 0).sum())


CASES = [("C2", "ip", None), ("C2", "up", None), ("C2", "3i", "gqe"), ("C2", "pi", "distmult-m"),
         ("C2", "ip", "complex-m"), ("C2", "2u", "rotate-m"),
         ("C3-rotate", "1p", None), ("C3-complex", "1p", None), ("C4", "2i", None), ("C4", "pni", None),
         ("C4", "up", None), ("C5-q2b", "pi", None), ("C5-q2b", "2u", None), ("C5-betae", "ip", None)]


@pytest.mark.parametrize("wl,structure,kind", CASES)
def test_full_size_step(wl, structure, kind):
    """kind: another model on the workload's shapes (GQE / -m variants have no config of their own)."""
    from paper_2110_14890_b200 import KGModel
    w = kggen.WORKLOADS[wl]
    cfg = w.model_config()
    if kind:
        cfg = kggen.ModelConfig(kind, w.dim, w.n_entities, w.n_relations)
    if wl.startswith("C5"):
        cfg.n_entities = kggen.shard_rows(w.n_entities, 8)   # the per-GPU shard bench.py trains
    M, K = w.M, w.K
    gm = KGModel(cfg, M, K)
    gm.init_params(5)
    gm.set_apply(True, keep_grads=True)
    table = oracle.SparseTable(cfg, 5)
    b, redrawn, masked = well_conditioned_batch(cfg, table, structure, M, K, seed=3)
    print(f"{wl} {structure}: {redrawn} queries re-drawn, {masked} near-tie DNF pairs masked out")
    lr = 1e-3
    assert redrawn <= 0.1 * M, f"{redrawn} of {M} queries re-drawn"
    # (before oracle_step: it applies the update to `table`)
    allow = q2b_flip_allowance(cfg, table, b, M, K) if cfg.kind == "q2b" else None
    ta_rows, ta_dense, n_dec = traced_flip_allowance(cfg, table, b, M, K)
    ref = oracle.oracle_step(cfg, table, [b], lr, apply=True)
    if allow is not None:
        allow_rows, allow_dense, n_terms = allow
    else:
        allow_rows, allow_dense, n_terms = np.zeros_like(ref.grad_rows), np.zeros_like(ref.grad_dense), 0
    allow_rows = allow_rows + ta_rows
    allow_dense = allow_dense + ta_dense
    info = gm.step(gm.host_batch(b), lr)
    g = gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K)
    assert abs(info.loss - ref.loss) <= RTOL * abs(ref.loss), (info.loss, ref.loss)
    assert_close(g["d_pos"], ref.d_pos[0], what="D+")
    assert_close(g["d_neg"], ref.d_neg[0], what="D")
    np.testing.assert_array_equal(g["uniq"], ref.uniq)
    assert info.n_touched == len(ref.uniq)
    n1, a1 = assert_close_allow(g["grad_rows"], ref.grad_rows, "dL/dtheta_E rows", allow_rows)
    n2, a2 = assert_close_allow(g["grad_dense"], ref.grad_dense, "dL/dtheta_D", allow_dense)
    print(f"{wl} {structure}: {n_dec} ReLU / clamp decisions within 2e-6 of their kink")
    print(f"{wl} {structure}: {n_terms} terms within 1e-6 of a kink; elements with an allowance: rows {a1} of "
          f"{allow_rows.size}, dense {a2} of {allow_dense.size}; beyond the plain bound: rows {n1}, dense {n2}")
    # after the step: an element whose gradient carries a flip allowance may take another Adam
    # step (at t = 1 the update is ~ -lr sign(g)); those are checked through the gradients above
    keep = (np.abs(ref.m_new) >= 1e-4 * np.abs(ref.m_new).max()) & (allow_rows <= 0.1 * np.abs(ref.grad_rows))
    assert_close(gm.read_rows(ref.uniq), ref.rows_new, what="theta_E rows after the step", mask=keep)
    keepd = (np.abs(ref.dense_m_new) >= 1e-4 * np.abs(ref.dense_m_new).max()) & (allow_dense <= 0.1 * np.abs(ref.grad_dense))
    assert_close(gm.read_dense(0), ref.dense_new, what="theta_D after the step", mask=keepd)
    gm.close()


UNCONDITIONED = [("C5-q2b", "pi"), ("C5-q2b", "3i"), ("C5-betae", "ip"), ("C4", "2in")]


@pytest.mark.parametrize("wl,structure", UNCONDITIONED)
def test_full_size_forward_unconditioned(wl, structure):
    """The seeded batch exactly as bench.py draws it (no re-drawn queries, no masked pairs): the
    forward outputs -- every D+ and D_ij and the loss -- are continuous in the fp32 rounding of
    every discrete decision the forward takes (ReLU, clamp, min), so they meet the plain 1e-5 bar
    with no conditioning; the touched-row set is bit-exact."""
    from paper_2110_14890_b200 import KGModel
    w = kggen.WORKLOADS[wl]
    cfg = w.model_config()
    if wl.startswith("C5"):
        cfg.n_entities = kggen.shard_rows(w.n_entities, 8)
    M, K = w.M, w.K
    gm = KGModel(cfg, M, K)
    gm.init_params(7)
    gm.set_apply(False, keep_grads=True)
    table = oracle.SparseTable(cfg, 7)
    b = kggen.make_batch(cfg, structure, M, K, seed=11, step=0)
    ref = oracle.oracle_step(cfg, table, [b], 1e-3, apply=False)
    info = gm.step(gm.host_batch(b), 1e-3)
    g = gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K)
    assert abs(info.loss - ref.loss) <= RTOL * abs(ref.loss), (info.loss, ref.loss)
    assert_close(g["d_pos"], ref.d_pos[0], what="D+")
    assert_close(g["d_neg"], ref.d_neg[0], what="D")
    np.testing.assert_array_equal(g["uniq"], ref.uniq)
    gm.close()
