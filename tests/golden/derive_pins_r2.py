"""Derive tests/golden/pins_r2.json -- hand-set worked examples that fix the parts of the
oracle which the paper defines but round 1 left unpinned (DNF min, the Q2B intersection,
the Q2B projection ReLU, Eq. 1's 1/|N_q|, the structure slot wiring and the negated branch,
the BetaE projection's +1 / clamp).

This script does NOT import oracle/ or the CUDA path.  It evaluates every example with
operator weights chosen so that each operator of Table 1 collapses to a
closed form a reader can check by hand:

  GQE   (d = 2)  P(q, r) = q + r;  DeepSet with W1 = W2 = I, b = 0:  I({q_i}) = mean_i ReLU(q_i);
                 D = ||q - v||_2                                    (Table 1, A2, A4)
  Q2B   (d = 2)  P((c, o), r) = (c + r_c, o + ReLU(r_o))            (A6)
                 attention with W1 = W2 = I, b = 0: a_i = softmax_i ReLU(c_i) per dimension,
                 c = sum_i a_i c_i;  offset DeepSet with V1 = V2 = I, e = 0:
                 o = min_i o_i * sigmoid(mean_i ReLU(o_i))           (A4, A5)
                 D = sum ReLU(|v - c| - o) + alpha sum min(|v - c|, o)   (A7)
  BetaE (d = 4)  e(x) = clamp(x + 1, 0.05, 1e9)                      (A8)
                 MLP with H = 2d, W1 = I, W2 = I, W0 = [2I | I], b = 0:
                 P(q, y) = clamp(2 q + ReLU(y) + 1, 0.05, 1e9)       (A9; non-commutative
                 in the order of the relations, so chain order is observable)
                 attention with U1 = I, U2 = [I | 0], c = 0: w_i = softmax_i(alpha_i) per dimension,
                 I = (sum w_i alpha_i, sum w_i beta_i)               (A5)
                 N(q) = 1/q                                          (A25)
                 D = sum_k KL(Beta(e(v)_k) || Beta(q_k)), entity first (A10), with scipy's
                 gammaln / digamma
  union          DNF: D = min over disjuncts                          (Def. 1, A11)
  loss           Eq. 1 P:L177-180 with n_i = popcount(mask row i)     (A12)

The structure DAGs are written from SURVEY App. A.3 and reading A25 (slots in execution
order, A21).  For each example the script also checks the example's POWER: every other
wiring (each permutation of the relation slots and of the anchor slots; for the negation
structures the negation moved to each other intersection input, or dropped) must change
D+ or D- by more than 1e-6 relative -- unless the change is a symmetry of the structure
(equal on three random draws, e.g. swapping the two branches of a 2i).  A seed whose
example cannot tell some wiring apart is rejected and the next seed is tried.

    python tests/golden/derive_pins_r2.py      (rewrites tests/golden/pins_r2.json)
"""
import itertools
import json
import math
import os

import numpy as np
from scipy.special import digamma, gammaln

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pins_r2.json")
ALPHA = 0.02   # Q2B alpha (A7)


def relu(x):
    return np.maximum(x, 0.0)


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def softplus(z):
    return math.log1p(math.exp(-abs(z))) + max(z, 0.0)


# ------------------------------------------------------------------ structures (App. A.3, A25)
# ('a', slot) | ('p', child, rel_slot) | ('i', [children]) | ('u', [children]) | ('n', child)
def A(s):
    return ("a", s)


def P(c, s):
    return ("p", c, s)


def I(*cs):
    return ("i", list(cs))


def U(*cs):
    return ("u", list(cs))


def N(c):
    return ("n", c)


STRUCT = {
    "1p": P(A(0), 0),
    "2p": P(P(A(0), 0), 1),
    "3p": P(P(P(A(0), 0), 1), 2),
    "2i": I(P(A(0), 0), P(A(1), 1)),
    "3i": I(P(A(0), 0), P(A(1), 1), P(A(2), 2)),
    "ip": P(I(P(A(0), 0), P(A(1), 1)), 2),
    "pi": I(P(P(A(0), 0), 1), P(A(1), 2)),
    "2u": U(P(A(0), 0), P(A(1), 1)),
    "up": P(U(P(A(0), 0), P(A(1), 1)), 2),
    "2in": I(P(A(0), 0), N(P(A(1), 1))),
    "3in": I(P(A(0), 0), P(A(1), 1), N(P(A(2), 2))),
    "inp": P(I(P(A(0), 0), N(P(A(1), 1))), 2),
    "pin": I(P(P(A(0), 0), 1), N(P(A(1), 2))),
    "pni": I(N(P(P(A(0), 0), 1)), P(A(1), 2)),
}
N_ANCHORS = {"1p": 1, "2p": 1, "3p": 1, "2i": 2, "3i": 3, "ip": 2, "pi": 2, "2u": 2, "up": 2,
             "2in": 2, "3in": 3, "inp": 2, "pin": 2, "pni": 2}
N_RELS = {"1p": 1, "2p": 2, "3p": 3, "2i": 2, "3i": 3, "ip": 3, "pi": 3, "2u": 2, "up": 3,
          "2in": 2, "3in": 3, "inp": 3, "pin": 3, "pni": 3}


def negation_variants(t):
    """Trees with the negation moved to another input of its intersection, or dropped."""
    out = []

    def strip(x):
        return x[1] if x[0] == "n" else x

    def walk(x, rebuild):
        if x[0] == "i" and any(c[0] == "n" for c in x[1]):
            base = [strip(c) for c in x[1]]
            out.append(rebuild(("i", base)))                        # negation dropped
            for k in range(len(base)):
                cs = list(base)
                cs[k] = ("n", cs[k])
                if cs != x[1]:
                    out.append(rebuild(("i", cs)))                  # another input negated
            return
        if x[0] == "p":
            walk(x[1], lambda y: rebuild(("p", y, x[2])))
        elif x[0] in ("i", "u"):
            for k, c in enumerate(x[1]):
                walk(c, lambda y, k=k: rebuild((x[0], x[1][:k] + [y] + x[1][k + 1:])))
        elif x[0] == "n":
            walk(x[1], lambda y: rebuild(("n", y)))

    walk(t, lambda y: y)
    return out


# ------------------------------------------------------------------ models
class GQE:
    kind, dim = "gqe", 2

    def anchor(self, x):
        return x

    def project(self, q, r):
        return q + r["rel"]

    def intersect(self, qs):
        return np.mean([relu(q) for q in qs], axis=0)

    def dist(self, q, v):
        return float(np.linalg.norm(q - v))


class Q2B:
    kind, dim = "q2b", 2

    def anchor(self, x):
        return np.concatenate([x, np.zeros_like(x)])

    def project(self, q, r):
        d = self.dim
        return np.concatenate([q[:d] + r["rel_center"], q[d:] + relu(r["rel_offset"])])

    def intersect(self, qs):
        d = self.dim
        C = np.array([q[:d] for q in qs])
        O = np.array([q[d:] for q in qs])
        logits = relu(C)
        a = np.exp(logits) / np.exp(logits).sum(axis=0)
        return np.concatenate([(a * C).sum(axis=0), O.min(axis=0) * sigmoid(relu(O).mean(axis=0))])

    def dist(self, q, v):
        d = self.dim
        delta = np.abs(v - q[:d])
        o = q[d:]
        return float(relu(delta - o).sum() + ALPHA * np.minimum(delta, o).sum())


class BetaE:
    kind, dim = "betae", 4

    def e(self, x):
        return np.clip(x + 1.0, 0.05, 1e9)

    def anchor(self, x):
        return self.e(x)

    def project(self, q, r):
        return np.clip(2.0 * q + relu(r["rel"]) + 1.0, 0.05, 1e9)

    def intersect(self, qs):
        m = self.dim // 2
        Al = np.array([q[:m] for q in qs])
        Be = np.array([q[m:] for q in qs])
        w = np.exp(Al) / np.exp(Al).sum(axis=0)
        return np.concatenate([(w * Al).sum(axis=0), (w * Be).sum(axis=0)])

    def negate(self, q):
        return 1.0 / q

    def dist(self, q, v):
        m = self.dim // 2
        ev = self.e(v)
        a1, b1, a2, b2 = ev[:m], ev[m:], q[:m], q[m:]
        lnB = lambda a, b: gammaln(a) + gammaln(b) - gammaln(a + b)
        kl = (lnB(a2, b2) - lnB(a1, b1) + (a1 - a2) * digamma(a1) + (b1 - b2) * digamma(b1)
              + (a2 - a1 + b2 - b1) * digamma(a1 + b1))
        return float(kl.sum())


def evaluate(model, tree, anchors, rels):
    """DNF disjunct embeddings of a structure tree (unions expanded, A11)."""
    def ev(x):
        if x[0] == "a":
            return [model.anchor(anchors[x[1]])]
        if x[0] == "p":
            return [model.project(q, rels[x[2]]) for q in ev(x[1])]
        if x[0] == "n":
            return [model.negate(q) for q in ev(x[1])]
        if x[0] == "u":
            return [q for c in x[1] for q in ev(c)]
        if x[0] == "i":
            parts = [ev(c) for c in x[1]]
            assert all(len(p) == 1 for p in parts), "no union below an intersection in these DAGs"
            return [model.intersect([p[0] for p in parts])]
        raise ValueError(x)
    return ev(tree)


def distances(model, tree, anchors, rels, v_pos, v_neg):
    qs = evaluate(model, tree, anchors, rels)
    return min(model.dist(q, v_pos) for q in qs), min(model.dist(q, v_neg) for q in qs)


# ------------------------------------------------------------------ parameter draws
def draw(model, rng, na, nr):
    d = model.dim
    g = lambda *shape: np.round(rng.uniform(-1.0, 1.0, size=shape) * 8) / 8      # multiples of 1/8
    if model.kind == "betae":
        anchors = [np.round(rng.uniform(-0.5, 1.5, size=d) * 8) / 8 for _ in range(na)]
        rels = [{"rel": g(d)} for _ in range(nr)]
        v_pos = np.round(rng.uniform(0.5, 6.0, size=d) * 8) / 8
        v_neg = np.round(rng.uniform(0.5, 6.0, size=d) * 8) / 8
    elif model.kind == "q2b":
        anchors = [2 * g(d) for _ in range(na)]
        rels = [{"rel_center": 2 * g(d), "rel_offset": g(d)} for _ in range(nr)]
        v_pos, v_neg = 3 * g(d), 3 * g(d)
    else:
        anchors = [2 * g(d) for _ in range(na)]
        rels = [{"rel": 2 * g(d)} for _ in range(nr)]
        v_pos, v_neg = 3 * g(d), 3 * g(d)
    return anchors, rels, v_pos, v_neg


def alternatives(structure):
    """(label, tree, anchor permutation, relation permutation) of every other wiring."""
    t = STRUCT[structure]
    na, nr = N_ANCHORS[structure], N_RELS[structure]
    out = []
    for pa in itertools.permutations(range(na)):
        for pr in itertools.permutations(range(nr)):
            if pa != tuple(range(na)) or pr != tuple(range(nr)):
                out.append((f"anchors {pa} relations {pr}", t, pa, pr))
    for k, tv in enumerate(negation_variants(t)):
        out.append((f"negation variant {k}", tv, tuple(range(na)), tuple(range(nr))))
    return out


def pair(model, tree, anchors, rels, v_pos, v_neg, pa, pr):
    return distances(model, tree, [anchors[i] for i in pa], [rels[i] for i in pr], v_pos, v_neg)


def differs(x, y, rel=1e-6):
    return any(abs(a - b) > rel * max(abs(a), abs(b), 1e-3) for a, b in zip(x, y))


def structure_example(model, structure, seed0):
    na, nr = N_ANCHORS[structure], N_RELS[structure]
    tree = STRUCT[structure]
    ident_a, ident_r = tuple(range(na)), tuple(range(nr))
    alts = alternatives(structure)
    # symmetries: alternatives equal to the true wiring on three random draws
    sym = set()
    for label, t2, pa, pr in alts:
        same = True
        for k in range(3):
            rng = np.random.default_rng(10_000 + k)
            an, rl, vp, vn = draw(model, rng, na, nr)
            an = [x + rng.normal(size=x.shape) * 0.01 for x in an]
            if differs(pair(model, tree, an, rl, vp, vn, ident_a, ident_r),
                       pair(model, t2, an, rl, vp, vn, pa, pr), 1e-12):
                same = False
                break
        if same:
            sym.add(label)
    for seed in range(seed0, seed0 + 500):
        rng = np.random.default_rng(seed)
        an, rl, vp, vn = draw(model, rng, na, nr)
        ref = pair(model, tree, an, rl, vp, vn, ident_a, ident_r)
        if model.kind == "betae" and not all(3.0 < x < 60.0 for x in ref):
            continue      # keep the Eq. 1 terms away from saturation
        if model.kind != "betae" and not all(0.2 < x for x in ref):
            continue
        if all(differs(ref, pair(model, t2, an, rl, vp, vn, pa, pr))
               for label, t2, pa, pr in alts if label not in sym):
            return dict(seed=seed, anchors=[x.tolist() for x in an],
                        relations=[{k: v.tolist() for k, v in r.items()} for r in rl],
                        positive=vp.tolist(), negative=vn.tolist(), d_pos=ref[0], d_neg=ref[1],
                        symmetries=sorted(sym),
                        n_alternatives_distinguished=len(alts) - len(sym))
    raise RuntimeError(f"no distinguishing example for {model.kind} {structure}")


GAMMA = {"gqe": 2.0, "q2b": 2.0, "betae": 12.0}


def loss_one(d_pos, d_neg, gamma):
    """Eq. 1 for one query with one masked-in negative (n = 1)."""
    return softplus(d_pos - gamma) + softplus(gamma - d_neg)


def union_gradient_example():
    """2u / up with distinct branches (GQE): D = min over disjuncts and the gradient flows
    only into the argmin disjunct (Def. 1, A11).  Hand-set so that the positive is
    nearest to disjunct 0 and the negative to disjunct 1.
      2u: q0 = a0 + r0 = (1, 0), q1 = a1 + r1 = (0, 3)
      up: q0 = a0 + r0 + r2 = (1, 0), q1 = a1 + r1 + r2 = (0, 3)  (r2 shared)
      v+ = (1, 1): D(q0) = 1, D(q1) = sqrt 5      -> D+ = 1 via disjunct 0
      v- = (0, 4): D(q0) = sqrt 17, D(q1) = 1     -> D- = 1 via disjunct 1
      gamma = 1, M = K = n = 1: dl/dD+ = sigma(0) = 1/2, dl/dD- = -sigma(0) = -1/2
      grad a0 = grad r0 = 1/2 (q0 - v+)/1 = (0, -1/2);  grad v+ = (0, 1/2)
      grad a1 = grad r1 = -1/2 (q1 - v-)/1 = (0, 1/2);  grad v- = (0, -1/2)
      up: grad r2 = grad r0 + grad r1 = (0, 0)"""
    ex = {}
    for s, a, r in (("2u", [[0.0, 0.0], [0.0, 1.0]], [[1.0, 0.0], [0.0, 2.0]]),
                    ("up", [[0.0, 0.0], [0.0, 1.0]], [[2.0, -1.0], [1.0, 1.0], [-1.0, 1.0]])):
        q = [np.array(a[0]) + np.array(r[0]), np.array(a[1]) + np.array(r[1])]
        if s == "up":
            q = [x + np.array(r[2]) for x in q]
        assert np.allclose(q[0], [1, 0]) and np.allclose(q[1], [0, 3])
        vp, vn = np.array([1.0, 1.0]), np.array([0.0, 4.0])
        dp = [np.linalg.norm(x - vp) for x in q]
        dn = [np.linalg.norm(x - vn) for x in q]
        kp, kn = int(np.argmin(dp)), int(np.argmin(dn))
        gp, gn = sigmoid(min(dp) - 1.0), -sigmoid(1.0 - min(dn))
        ga = [np.zeros(2), np.zeros(2)]
        ga[kp] += gp * (q[kp] - vp) / dp[kp]
        ga[kn] += gn * (q[kn] - vn) / dn[kn]
        grel = [ga[0].copy(), ga[1].copy()] + ([ga[0] + ga[1]] if s == "up" else [])
        ex[s] = dict(gamma=1.0, anchors=a, relations=r, positive=vp.tolist(), negative=vn.tolist(),
                     d_pos=min(dp), d_neg=min(dn), loss=loss_one(min(dp), min(dn), 1.0),
                     d_pos_max=max(dp), d_neg_max=max(dn),
                     grad_anchors=[x.tolist() for x in ga], grad_relations=[x.tolist() for x in grel],
                     grad_positive=(-gp * (q[kp] - vp) / dp[kp]).tolist(),
                     grad_negative=(-gn * (q[kn] - vn) / dn[kn]).tolist())
    return ex


def partial_mask_example():
    """Eq. 1 on a partially masked pool (P:L177-180 with Mask of P:L389, A12): GQE 1p, d = 2,
    gamma = 2, M = 2, K = 3, the relation row 0 so q_i = anchor_i.
      q0 = (0, 0), q1 = (0, 0.5); v+ = (1, 0) for both; pool v_j = (0, j + 1)
      mask row 0 = (1, 0, 1) -> n_0 = 2; mask row 1 = (0, 1, 1) -> n_1 = 2
      l_i = softplus(D+_i - 2) + (1/n_i) sum_j mask_ij softplus(2 - D_ij); L = (l_0 + l_1)/2
      dL/dv_j = sum_i -mask_ij sigmoid(2 - D_ij) / (n_i M) * (v_j - q_i)/D_ij"""
    gamma, M = 2.0, 2
    q = [np.array([0.0, 0.0]), np.array([0.0, 0.5])]
    vp = np.array([1.0, 0.0])
    pool = [np.array([0.0, j + 1.0]) for j in range(3)]
    mask = [[1, 0, 1], [0, 1, 1]]
    loss = 0.0
    gpool = [np.zeros(2) for _ in range(3)]
    for i in range(M):
        n = sum(mask[i])
        dp = np.linalg.norm(q[i] - vp)
        li = softplus(dp - gamma)
        for j in range(3):
            if mask[i][j]:
                D = np.linalg.norm(q[i] - pool[j])
                li += softplus(gamma - D) / n
                gpool[j] += -sigmoid(gamma - D) / (n * M) * (pool[j] - q[i]) / D
        loss += li / M
    return dict(gamma=gamma, queries=[x.tolist() for x in q], positive=vp.tolist(),
                pool=[x.tolist() for x in pool], mask=mask, loss=loss, grad_pool=[x.tolist() for x in gpool])


def main():
    out = {
        "_about": ("Worked examples with hand-set operator weights, derived by tests/golden/derive_pins_r2.py "
                   "(plain numpy + scipy.special; it never imports oracle/ or the CUDA path). See that "
                   "script's docstring for the closed form of every operator and the citation of each."),
        "union_gradient": union_gradient_example(),
        "partial_mask": partial_mask_example(),
        "betae_projection_zero_mlp": {
            "citation": "Table 1 P:L143 MLP(Em(q), Em(r)); readings A8 (clamp(x + 1, 0.05, 1e9)), A9",
            "derivation": "W1 = W2 = W0 = 0, b1 = b2 = 0 => P(q, r) = clamp(b0 + 1, 0.05, 1e9)",
            "b0": [0.25, -2.0, 5.0, -0.5], "out": [1.25, 0.05, 6.0, 0.5]},
        "q2b_projection_relu": {
            "citation": "Table 1 P:L140 Em(q)+Em(r) on boxes; reading A6 (offset grows by ReLU(r_o))",
            "derivation": "anchor (c, o) = ((0.5, -1), (0, 0)); r_c = (1, 1), r_o = (-1, 2) => q = ((1.5, 0), (0, 2)); "
                          "v = (2.5, 0.5): |v - c| = (1, 0.5); D = ReLU(1 - 0) + ReLU(0.5 - 2) + 0.02 (0 + 0.5) = 1.01",
            "anchor": [0.5, -1.0], "rel_center": [1.0, 1.0], "rel_offset": [-1.0, 2.0], "v": [2.5, 0.5],
            "dist": 1.01},
        "structures": {},
    }
    for model in (GQE(), Q2B(), BetaE()):
        structs = list(STRUCT) if model.kind == "betae" else [s for s in STRUCT if "n" not in s]
        for s in structs:
            ex = structure_example(model, s, 1)
            ex["gamma"] = GAMMA[model.kind]
            ex["loss"] = loss_one(ex["d_pos"], ex["d_neg"], ex["gamma"])
            out["structures"][f"{model.kind}:{s}"] = ex
            print(model.kind, s, "seed", ex["seed"], "D+", ex["d_pos"], "D-", ex["d_neg"],
                  "alternatives told apart", ex["n_alternatives_distinguished"], "symmetries", ex["symmetries"])
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
