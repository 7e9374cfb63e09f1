"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds the *input format* and the *input recipe* only -- none of the
method's arithmetic (no projection, intersection, distance, loss, gradient or
optimizer code lives here).  Both `oracle/` (test infrastructure) and the
product binding read their inputs from here, so that a parity test compares the
two implementations on byte-identical inputs.

Contents
  * query-structure shapes (anchor / relation slot counts, SURVEY App. A.3,
    PAPER.md P:L490 "the same 14 query structures proposed in BetaE"; the 9
    non-negation ones are built here),
  * the dense-parameter layout theta_D (§4.1: theta_E is the
    entity matrix, theta_D = theta \\ theta_E),
  * a counter-based uniform generator used for parameter init (DESIGN.md
    reading R-init): value = f(seed, stream, index); the CUDA init kernel
    implements the same function, so neither side ever needs the other's
    output,
  * the batch recipe of DESIGN.md §"Input recipe" (Zipf anchors/answers,
    uniform pool with replacement P:L222, Bernoulli mask P:L389),
  * the BASELINE.json config presets C1-C5.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

# --------------------------------------------------------------------------
# Model kinds and structures (ids match include/kg.h)
# --------------------------------------------------------------------------
MODELS = ["gqe", "q2b", "betae", "transe", "rotate", "distmult", "complex",
          "rotate-m", "distmult-m", "complex-m"]     # App. B P:L629-638 multi-hop extensions (f4)
MODEL_ID = {m: i for i, m in enumerate(MODELS)}
SINGLE_HOP = {"transe", "rotate", "distmult", "complex"}
M_VARIANTS = {"rotate-m": "rotate", "distmult-m": "distmult", "complex-m": "complex"}

STRUCTURES = ["1p", "2p", "3p", "2i", "3i", "ip", "pi", "2u", "up"]
# the 5 structures with negation (Table 10; BetaE only, Table 1 'Negation' column)
NEG_STRUCTURES = ["2in", "3in", "inp", "pin", "pni"]
ALL_STRUCTURES = STRUCTURES + NEG_STRUCTURES
STRUCTURE_ID = {s: i for i, s in enumerate(ALL_STRUCTURES)}
# slot counts per structure (execution order A21)
N_ANCHORS = {"1p": 1, "2p": 1, "3p": 1, "2i": 2, "3i": 3, "ip": 2, "pi": 2, "2u": 2, "up": 2,
             "2in": 2, "3in": 3, "inp": 2, "pin": 2, "pni": 2}
N_RELS = {"1p": 1, "2p": 2, "3p": 3, "2i": 2, "3i": 3, "ip": 3, "pi": 3, "2u": 2, "up": 3,
          "2in": 2, "3in": 3, "inp": 3, "pin": 3, "pni": 3}

# Default margins (reading A14; the paper states no value).
DEFAULT_GAMMA = {"gqe": 24.0, "q2b": 24.0, "betae": 60.0, "transe": 24.0,
                 "rotate": 24.0, "distmult": 24.0, "complex": 24.0,
                 "rotate-m": 24.0, "distmult-m": 24.0, "complex-m": 24.0}


@dataclass
class ModelConfig:
    kind: str
    dim: int
    n_entities: int
    n_relations: int
    gamma: float = None
    box_alpha: float = 0.02          # Q2B alpha (A7)
    hidden: int = None               # BetaE projection MLP width (A9), default 4*dim
    beta1: float = 0.9               # Adam (A15)
    beta2: float = 0.999
    eps: float = 1e-8

    def __post_init__(self):
        if self.gamma is None:
            self.gamma = DEFAULT_GAMMA[self.kind]
        if self.hidden is None:
            self.hidden = 4 * self.dim

    @property
    def rho(self) -> float:
        """Init half-range of entity/relation rows (A23): (gamma + 2) / d."""
        return (self.gamma + 2.0) / self.dim


# --------------------------------------------------------------------------
# theta_D layout: ordered segments (name, shape, lo, hi)
# --------------------------------------------------------------------------
def dense_layout(cfg: ModelConfig):
    """Ordered list of (name, shape, init_lo, init_hi) making up theta_D.

    Weights are stored row-major [out][in] (y = W x + b).  Every segment size is
    a multiple of 4 floats when dim % 8 == 0 and hidden % 8 == 0.
    """
    d, R, H = cfg.dim, cfg.n_relations, cfg.hidden
    m = d // 2
    rho = cfg.rho
    w = 1.0 / math.sqrt(d)
    k = M_VARIANTS.get(cfg.kind, cfg.kind)   # an -m variant keeps its base model's relation table
    segs = []
    if k in ("gqe", "transe", "distmult", "complex"):
        segs.append(("rel", (R, d), -rho, rho))
    elif k == "q2b":
        segs.append(("rel_center", (R, d), -rho, rho))
        segs.append(("rel_offset", (R, d), 0.0, rho))
    elif k == "betae":
        segs.append(("rel", (R, d), -rho, rho))
    elif k == "rotate":
        segs.append(("rel_phase", (R, m), -math.pi, math.pi))
    else:
        raise ValueError(k)
    if k == "gqe" or cfg.kind in M_VARIANTS:   # DeepSet intersection (A4; GQE, and the -m variants P:L632)
        segs += [("ds_W1", (d, d), -w, w), ("ds_b1", (d,), -w, w),
                 ("ds_W2", (d, d), -w, w), ("ds_b2", (d,), -w, w)]
    elif k == "q2b":      # center attention (A5) + offset DeepSet (A4)
        segs += [("att_W1", (d, d), -w, w), ("att_b1", (d,), -w, w),
                 ("att_W2", (d, d), -w, w), ("att_b2", (d,), -w, w),
                 ("off_W1", (d, d), -w, w), ("off_b1", (d,), -w, w),
                 ("off_W2", (d, d), -w, w), ("off_b2", (d,), -w, w)]
    elif k == "betae":    # projection MLP (A9) + attention (A5)
        w1 = 1.0 / math.sqrt(2 * d)
        wh = 1.0 / math.sqrt(H)
        segs += [("prj_W1", (H, 2 * d), -w1, w1), ("prj_b1", (H,), -w1, w1),
                 ("prj_W2", (H, H), -wh, wh), ("prj_b2", (H,), -wh, wh),
                 ("prj_W0", (d, H), -wh, wh), ("prj_b0", (d,), -wh, wh),
                 ("att_U1", (d, d), -w, w), ("att_c1", (d,), -w, w),
                 ("att_U2", (m, d), -w, w), ("att_c2", (m,), -w, w)]
    return segs


def dense_offsets(cfg: ModelConfig):
    """name -> (offset, shape) in the flat theta_D array, and the total size."""
    off = 0
    out = {}
    for name, shape, _, _ in dense_layout(cfg):
        n = int(np.prod(shape))
        out[name] = (off, shape)
        off += n
    return out, off


# --------------------------------------------------------------------------
# Counter-based generator (splitmix64 finaliser).  The CUDA init kernel in
# csrc/k_adam.cu implements the same function (tests compare bit-exactly).
# --------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G1 = np.uint64(0x9E3779B97F4A7C15)
_G2 = np.uint64(0xD1B54A32D192ED03)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, stream: int, idx, lo: float, hi: float) -> np.ndarray:
    """float32 U[lo, hi) as a pure function of (seed, stream, idx).

    h = mix(mix(seed ^ stream*G1) + idx*G2);  u = (h >> 40) * 2^-24 (exact in fp32);
    x = fl32(lo) + fl32(fl32(hi) - fl32(lo)) * u   (each op rounded once, no FMA).
    """
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = _mix64(np.uint64(seed) ^ (np.uint64(stream) * _G1))
        h = _mix64(s + idx * _G2)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    lo32 = np.float32(lo)
    span = np.float32(np.float32(hi) - lo32)
    prod = (span * u).astype(np.float32)
    return (lo32 + prod).astype(np.float32)


ENTITY_STREAM = 0


def init_entity_rows(cfg: ModelConfig, seed: int, ids) -> np.ndarray:
    """Initial theta_E rows (A23) for the given global entity ids: float32 [n, d]."""
    ids = np.asarray(ids, dtype=np.uint64).reshape(-1)
    d = cfg.dim
    flat = ids[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]
    return counter_uniform(seed, ENTITY_STREAM, flat, -cfg.rho, cfg.rho)


def init_dense(cfg: ModelConfig, seed: int) -> np.ndarray:
    """Initial theta_D (flat float32), segment s drawn from stream 1 + s."""
    parts = []
    for s, (name, shape, lo, hi) in enumerate(dense_layout(cfg)):
        n = int(np.prod(shape))
        parts.append(counter_uniform(seed, 1 + s, np.arange(n, dtype=np.uint64), lo, hi))
    return np.concatenate(parts).astype(np.float32)


# --------------------------------------------------------------------------
# Batch recipe
# --------------------------------------------------------------------------
def _affine_perm(k: np.ndarray, n: int, salt: int) -> np.ndarray:
    """Bijection of [0, n): k -> (k*A + B) mod n with gcd(A, n) = 1."""
    A = 2654435761  # prime
    while math.gcd(A, n) != 1:
        A += 2
    B = (salt * 40503) % max(n, 1)
    return ((k.astype(np.uint64) * np.uint64(A % n) + np.uint64(B)) % np.uint64(n)).astype(np.int64)


def zipf_ids(rng: np.random.Generator, size, n: int, s: float, salt: int) -> np.ndarray:
    """Bounded Zipf(s) ranks over [0, n) mapped through a fixed permutation."""
    size = int(np.prod(size))
    out = np.empty(size, dtype=np.int64)
    filled = 0
    while filled < size:
        if s > 1.0:
            k = rng.zipf(s, size=2 * (size - filled) + 16)
            k = k[k <= n]
        else:  # s == 1: inverse CDF on the (small) support
            p = 1.0 / np.arange(1, n + 1)
            k = rng.choice(n, size=size - filled, p=p / p.sum()) + 1
        take = min(len(k), size - filled)
        out[filled:filled + take] = k[:take] - 1
        filled += take
    return _affine_perm(out, n, salt)


def pack_mask(bits: np.ndarray) -> np.ndarray:
    """bool [M, K] -> uint32 [M, ceil(K/32)], bit (j % 32) of word j // 32 (LSB first)."""
    M, K = bits.shape
    W = (K + 31) // 32
    pad = np.zeros((M, W * 32), dtype=bool)
    pad[:, :K] = bits
    b = pad.reshape(M, W, 32).astype(np.uint64)
    words = (b << np.arange(32, dtype=np.uint64)[None, None, :]).sum(axis=2)
    return words.astype(np.uint32)


def unpack_mask(words: np.ndarray, K: int) -> np.ndarray:
    M, W = words.shape
    bits = (words[:, :, None].astype(np.uint64) >> np.arange(32, dtype=np.uint64)) & np.uint64(1)
    return bits.reshape(M, W * 32)[:, :K].astype(bool)


def make_batch(cfg: ModelConfig, structure: str, M: int, K: int, seed: int = 0,
               step: int = 0, rank: int = 0, mask_p: float = 0.999) -> dict:
    """One synthetic mini-batch (N, {(q_i, V_qi, A_qi)}, Mask) in the P:L389 format.

    anchors int64 [M, n_anchor], relations int32 [M, n_rel] (execution order A21),
    answers int64 [M], negatives int64 [K] (uniform with replacement),
    mask uint32 [M, ceil(K/32)] (bit = 1: pool entry j is a negative of query i;
    the positive is never marked, A20).
    """
    rng = np.random.default_rng([seed, rank, step, STRUCTURE_ID[structure]])
    na, nr = N_ANCHORS[structure], N_RELS[structure]
    n, R = cfg.n_entities, cfg.n_relations
    anchors = zipf_ids(rng, (M, na), n, 1.1, salt=1).reshape(M, na)
    answers = zipf_ids(rng, (M,), n, 1.1, salt=1)
    relations = zipf_ids(rng, (M, nr), R, 1.0, salt=2).reshape(M, nr).astype(np.int32)
    negatives = rng.integers(0, n, size=K, dtype=np.int64)
    bits = rng.random((M, K)) < mask_p
    bits &= negatives[None, :] != answers[:, None]
    return dict(structure=structure, anchors=anchors, relations=relations,
                answers=answers, negatives=negatives, mask=pack_mask(bits), K=K, M=M)


# --------------------------------------------------------------------------
# Synthetic knowledge graph (input of the online sampler)
# --------------------------------------------------------------------------
def powerlaw_ranks(rng: np.random.Generator, size: int, n: int, a: float) -> np.ndarray:
    """Ranks in [0, n) with P(k) ~ (k+1)^-a (continuous inverse CDF on [1, n+1), a != 1)."""
    u = rng.random(size)
    e = 1.0 - a
    x = (((n + 1.0) ** e - 1.0) * u + 1.0) ** (1.0 / e)
    return np.minimum(np.floor(x).astype(np.int64) - 1, n - 1)


def make_kg(n_entities: int, n_relations: int, n_edges: int, seed: int = 0, a: float = 0.8,
            dedup: bool = True) -> dict:
    """A seeded synthetic KG G = (V, E, R) shaped like Table 3.

    Heads and tails follow a power law over ranks (exponent `a`) mapped through two
    fixed affine permutations (heavy-tailed in- and out-degrees, hubs differ), relations
    are Zipf(1.0).  Duplicate triples are dropped, so |E| <= n_edges.  Returns
    dict(h int64 [E], r int32 [E], t int64 [E], n_entities, n_relations), triples sorted
    by (h, r, t).  dedup=False skips the sort (large benches): the triples keep their draw
    order and may repeat; the samplers' indices drop repeats themselves.  Input recipe
    only: no traversal, sampling or index structure here.
    """
    rng = np.random.default_rng([seed, 0x6B67])
    h = _affine_perm(powerlaw_ranks(rng, n_edges, n_entities, a), n_entities, salt=3)
    t = _affine_perm(powerlaw_ranks(rng, n_edges, n_entities, a), n_entities, salt=4)
    r = zipf_ids(rng, (n_edges,), n_relations, 1.0, salt=5)
    if not dedup:
        return dict(h=h, r=r.astype(np.int32), t=t, n_entities=int(n_entities), n_relations=int(n_relations))
    hr = h * np.int64(n_relations) + r
    order = np.lexsort((t, hr))
    hr, t = hr[order], t[order]
    keep = np.ones(len(t), dtype=bool)
    keep[1:] = (hr[1:] != hr[:-1]) | (t[1:] != t[:-1])
    hr, t = hr[keep], t[keep]
    return dict(h=(hr // n_relations).astype(np.int64), r=(hr % n_relations).astype(np.int32),
                t=t.astype(np.int64), n_entities=int(n_entities), n_relations=int(n_relations))


def split_kg(kg: dict, valid_frac: float = 0.06, test_frac: float = 0.07, seed: int = 0):
    """Random edge split into G_train, G_valid = train + valid, G_test = train + valid + test
    (App. E; fractions of Table 3's FB15k-237 split).  Returns three KG dicts."""
    rng = np.random.default_rng([seed, 0x5917])
    E = len(kg["h"])
    u = rng.random(E)
    tr = u >= valid_frac + test_frac
    va = u < valid_frac + test_frac
    te = u < test_frac

    def sub(m):
        return dict(h=kg["h"][m], r=kg["r"][m], t=kg["t"][m], n_entities=kg["n_entities"],
                    n_relations=kg["n_relations"])
    return sub(tr), sub(tr | (va & ~te)), sub(np.ones(E, bool))


# Table 3 shapes (training edges), for the sampler benches and tests
KG_SHAPES = {
    "FB15k-237": (14505, 237, 272115),
    "FB400k": (409829, 918, 1075837),
    "ogbl-wikikg2": (2500604, 535, 16109182),
    "Freebase": (86054151, 14824, 304727650),
}


# --------------------------------------------------------------------------
# BASELINE.json configs C1-C5
# --------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    kind: str
    dim: int
    n_entities: int
    n_relations: int
    structures: list
    M: int
    K: int
    hidden: int = None
    note: str = ""

    def model_config(self, **kw) -> ModelConfig:
        return ModelConfig(kind=self.kind, dim=self.dim, n_entities=self.n_entities,
                           n_relations=self.n_relations, hidden=self.hidden, **kw)


ALL9 = list(STRUCTURES)
WORKLOADS = {
    "C1": Workload("C1", "gqe", 32, 1000, 10, ["1p", "2i"], 64, 16,
                   note="synthetic KG 1k entities / 10 relations, GQE d32, 1p+2i, B64, K16"),
    "C2": Workload("C2", "q2b", 400, 14505, 237, ALL9, 512, 128,
                   note="FB15k-237-shaped Q2B d400, 9 structures, B512, K128"),
    "C3-rotate": Workload("C3-rotate", "rotate", 200, 2500604, 535, ["1p"], 1024, 1024,
                          note="ogbl-wikikg2-shaped single-hop RotatE d200, B1024, K1024"),
    "C3-complex": Workload("C3-complex", "complex", 200, 2500604, 535, ["1p"], 1024, 1024,
                           note="ogbl-wikikg2-shaped single-hop ComplEx d200, B1024, K1024"),
    "C4": Workload("C4", "betae", 400, 409829, 918, ALL9, 512, 1024, hidden=1600,
                   note="FB400k-shaped BetaE d400, 9 structures, B512, K1024"),
    "C5-q2b": Workload("C5-q2b", "q2b", 400, 86054151, 14824, ALL9, 512, 1024,
                       note="Freebase-shaped Q2B d400, 9 structures, B512, K1024"),
    "C5-betae": Workload("C5-betae", "betae", 400, 86054151, 14824, ALL9, 512, 1024, hidden=1600,
                         note="Freebase-shaped BetaE d400, 9 structures, B512, K1024"),
    # SURVEY §8(d) "bandwidth-shaped variant for H1": B = K = 4096 per GPU, so the sparse
    # gather / segment-reduce / sparse-Adam kernels move enough rows to be measured against HBM
    "C5-q2b-bw": Workload("C5-q2b-bw", "q2b", 400, 86054151, 14824, ALL9, 4096, 4096,
                          note="bandwidth-shaped Freebase Q2B d400, 9 structures, B4096, K4096"),
    "C4-bw": Workload("C4-bw", "betae", 400, 409829, 918, ALL9, 4096, 4096, hidden=1600,
                      note="bandwidth-shaped FB400k BetaE d400, 9 structures, B4096, K4096"),
}


def shard_rows(n_entities: int, world: int) -> int:
    """Rows per rank under cyclic sharding owner(id) = id % world."""
    return (n_entities + world - 1) // world
