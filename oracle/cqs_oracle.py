"""ORACLE for CQS-decomposed exact attention (Stream-CQSA, arXiv 2604.20819).

*** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module.  The product path (paper_2604_20819_b200/, libcqs)
never imports, links or executes anything under oracle/, and this module imports nothing from it.

Plain, slow, obviously-correct CPU code in float64 NumPy.  Every function cites the PAPER.md passage
it follows as P:<line>.  Where the paper is silent the DESIGN.md "Readings" table (R1..R18, mirroring
SURVEY.md §8c) fixes the choice; those readings are cited as R<n>.

Parts:
  O0  difference sets / interest sets ............ Appendix B
  O2  literal Algorithm 3 BuildSubseq ............. P:269-307 (+ canonical segments & plan bytes)
  O1  dense softmax attention (+ full-row lse) .... definition; "exactly the same result" P:8
  O3  literal Algorithm 1 (raw exp, Num/Den) ...... P:41-52
  O4  LSE form: per-task (O_i, lse_i) + LSE merge . P:240 (Den_i = exp(lse), Num_i = out*Den_i)
  O5  device-memory model (memory_model.py) ....... P:145-162 budget-driven uniform depth (R14)
  O6  backward: dense gradients + literal Alg. 2 .. P:87-128, Appendix D P:429-502 (NEXT-1)
  O7  hybrid scheduling: leaf rule + plan bytes ..... P:154-160 (NEXT-2, reading R20)
  O8  per-level interest sets (mixed c) ............ P:136 (NEXT-3, reading R21)

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Eq. 1 / Fig. 2 / Fig. 3 facts, brute-force pair
coverage, closed forms (N=1 -> O=V, Q=K=0 -> mean V), an independent pure-Python loop evaluation,
torch float64 SDPA, granularity invariance and negative controls; O6 against central finite
differences and dO = 0 / linearity-in-V cases.  No function here is "parity
unpinned".
"""
from __future__ import annotations

import itertools
import math
import struct
from dataclasses import dataclass, field

import numpy as np

# ------------------------------------------------------------------------------------------------
# O0. Interest sets = cyclic (c, l, 1) difference sets
# ------------------------------------------------------------------------------------------------

#: Appendix B table.  The l=12 row is printed but is NOT a difference set (DESIGN R18).
PAPER_TABLE = {
    3: (7, (0, 1, 3)),
    4: (13, (0, 1, 3, 9)),
    5: (21, (0, 1, 4, 14, 16)),
    6: (31, (0, 1, 3, 8, 12, 18)),
    7: (43, None),
    8: (57, (0, 1, 3, 13, 32, 36, 43, 52)),
    9: (73, (0, 1, 3, 7, 15, 31, 36, 54, 63)),
    10: (91, (0, 1, 3, 9, 27, 49, 56, 61, 77, 81)),
    11: (111, None),
    12: (133, (0, 1, 4, 12, 21, 26, 45, 68, 84, 96, 98, 126)),
}


def chunk_count_for(l: int) -> int:
    """c = l(l-1)+1 from the pair-count identity c*l(l-1)/2 = c(c-1)/2."""
    return l * (l - 1) + 1


def difference_multiset(offsets, c):
    """All (a - b) mod c over ordered pairs a != b of the set."""
    return [(a - b) % c for a in offsets for b in offsets if a != b]


def is_difference_set(offsets, c) -> bool:
    """(c, l, 1) difference set: every nonzero residue appears exactly once (lambda=1)."""
    offs = list(offsets)
    if len(set(offs)) != len(offs) or any(not (0 <= o < c) for o in offs):
        raise ValueError("offsets must be distinct and in [0, c)")
    d = difference_multiset(offs, c)
    return sorted(d) == list(range(1, c))


def interest_sets_with_prefix01(c, l):
    """Exhaustive search over sets (0, 1, a_2..a_{l-1}) (method of P:356, brute force)."""
    out = []
    for rest in itertools.combinations(range(2, c), l - 2):
        s = (0, 1) + rest
        if is_difference_set(s, c):
            out.append(s)
    return out


def paired_interest_set(offsets, c):
    """(0,1,a2..a_{l-1}) -> (0, 1, c+1-a_{l-1}, ..., c+1-a_2)."""
    a = list(offsets)
    assert a[0] == 0 and a[1] == 1
    return tuple([0, 1] + [c + 1 - x for x in reversed(a[2:])])


# ------------------------------------------------------------------------------------------------
# O2. Algorithm 3  BuildSubseq(N, c, itr, I)
# ------------------------------------------------------------------------------------------------

def balanced_chunk_layout(L: int, c: int):
    """(starts, ends) of c contiguous chunks of [0, L).  The paper does not give the
    remainder rule; reading R1: the first (L mod c) chunks get ceil(L/c) tokens."""
    if L < c:
        raise ValueError("L < c: a chunk would be empty (R10)")
    q, r = divmod(L, c)
    sizes = [q + 1 if u < r else q for u in range(c)]
    starts = [0]
    for s in sizes[:-1]:
        starts.append(starts[-1] + s)
    ends = [st + sz for st, sz in zip(starts, sizes)]
    return starts, ends


def indices_to_runs(idx):
    """IndicesToRuns: maximal half-open runs [s, e) covering a sorted index list."""
    runs = []
    for i in idx:
        i = int(i)
        if runs and runs[-1][1] == i:
            runs[-1][1] = i + 1
        else:
            runs.append([i, i + 1])
    return [tuple(r) for r in runs]


@dataclass
class Entry:
    """One subseq_entries element plus the intermediate histories of Alg. 3."""
    quorum: tuple
    token_ids: np.ndarray                # int64, local order
    label_history: list                  # per level t: chunk id of each local position
    chunks_history: list                 # per level t: (owner q_t, chunks in I order)
    group_runs: list = field(default_factory=list)   # deduplicated masked groups (list of runs)


def build_subseq_entry(N: int, c: int, I, quorum) -> Entry:
    """Algorithm 3 body for one quorum tuple i = (q_1..q_itr), literally."""
    return build_subseq_entry_levels(N, [(c, I)] * len(quorum), quorum)


def build_subseq_entry_levels(N: int, levels, quorum) -> Entry:
    """Algorithm 3 body with interest set levels[t] = (c_t, I_t) at iteration t ("different
    values of c ... can be used at each iteration"; reading R21 — every other step unchanged)."""
    token_ids = np.arange(N, dtype=np.int64)
    label_history, chunks_history = [], []
    for t, q_t in enumerate(quorum):
        c, I = levels[t]
        L = len(token_ids)
        starts, ends = balanced_chunk_layout(L, c)
        chunks = [(q_t + o) % c for o in I]                        # P:281 (ordered by I, R2)
        labels = np.empty(L, dtype=np.int64)
        for u in range(c):
            labels[starts[u]:ends[u]] = u
        gather_idx = np.concatenate([np.arange(starts[u], ends[u]) for u in chunks])
        for s in range(len(label_history)):
            label_history[s] = label_history[s][gather_idx]
        label_history.append(labels[gather_idx])
        token_ids = token_ids[gather_idx]
        chunks_history.append((q_t, chunks))
    group_runs = []
    for t in range(len(quorum)):
        owner, chunks = chunks_history[t]
        labels = label_history[t]
        for chunk in chunks:
            if chunk == owner:
                continue
            idx = np.nonzero(labels == chunk)[0]
            runs = indices_to_runs(idx)
            if runs:
                group_runs.append(runs)
    uniq = []                                                      # P:301 Unique (R5: first kept)
    for g in group_runs:
        if g not in uniq:
            uniq.append(g)
    return Entry(tuple(quorum), token_ids, label_history, chunks_history, uniq)


def quorum_tuples(c: int, itr: int):
    """All (q_1..q_itr) in {0..c-1}^itr, lexicographic, q_1 most significant (R3)."""
    return list(itertools.product(range(c), repeat=itr))


def build_subseq(N: int, c: int, itr: int, I):
    """BuildSubseq(N, c, itr, I) -> subseq_entries."""
    if not is_difference_set(I, c):
        raise ValueError("interest set is not a (c,l,1) difference set")
    if N < c ** itr:
        raise ValueError("N < c^itr (R10)")
    return [build_subseq_entry(N, c, I, qt) for qt in quorum_tuples(c, itr)]


def local_mask(entry: Entry) -> np.ndarray:
    """LocalMaskFromGroupRuns(|token_ids|, group_runs): 1 everywhere except G x G for every
    masked group G (multiplicative 0/1 mask, R6)."""
    L = len(entry.token_ids)
    M = np.ones((L, L), dtype=np.float64)
    for g in entry.group_runs:
        pos = np.concatenate([np.arange(s, e) for s, e in g])
        M[np.ix_(pos, pos)] = 0.0
    return M


# ---- canonical segments & plan bytes (the form the GPU planner must reproduce bit-exactly) -------

def entry_segments(entry: Entry):
    """Cut the entry into maximal segments: runs of local positions with consecutive global token
    ids and identical per-level codes, code_t = index of the position's level-t chunk in I order
    (R4: code 0 = owner q_t).  Returns [(global_start, length, codes_tuple)] in local order."""
    L = len(entry.token_ids)
    codes = np.zeros((L, len(entry.chunks_history)), dtype=np.int64)
    for t, (_, chunks) in enumerate(entry.chunks_history):
        lab = entry.label_history[t]
        for ci, ch in enumerate(chunks):
            codes[lab == ch, t] = ci
    # a new segment starts at position p > 0 iff the global id does not continue or a code changes
    brk = np.ones(L, dtype=bool)
    if L > 1:
        brk[1:] = (np.diff(entry.token_ids) != 1) | np.any(codes[1:] != codes[:-1], axis=1)
    starts = np.nonzero(brk)[0]
    ends = np.append(starts[1:], L)
    return [(int(entry.token_ids[p]), int(e - p), tuple(int(x) for x in codes[p]))
            for p, e in zip(starts, ends)]


def segment_kept_matrix(entry: Entry, segs):
    """kept[a][b] for segment blocks, derived from the literal group runs: block (a, b) is
    masked iff some masked group contains both segments.  Asserts every segment lies wholly inside
    or wholly outside each group (so the block mask is exact, no element-level masking needed)."""
    bounds = []
    p = 0
    for (_, ln, _) in segs:
        bounds.append((p, p + ln))
        p += ln
    member = np.zeros((len(entry.group_runs), len(segs)), dtype=bool)
    for gi, g in enumerate(entry.group_runs):
        for si, (s0, s1) in enumerate(bounds):
            inside = sum(max(0, min(e, s1) - max(s, s0)) for s, e in g)
            assert inside in (0, s1 - s0), "segment straddles a mask group"
            member[gi, si] = inside == s1 - s0
    n = len(segs)
    kept = np.ones((n, n), dtype=bool)
    for gi in range(len(entry.group_runs)):
        idx = np.nonzero(member[gi])[0]
        kept[np.ix_(idx, idx)] = False
    return kept


def entry_work(segs, kept) -> int:
    """Kept (query, key) pairs of the task = number of unmasked mask entries."""
    return int(sum(segs[a][1] * segs[b][1] for a in range(len(segs)) for b in range(len(segs))
                   if kept[a, b]))


PLAN_MAGIC = b"CQSP"
PLAN_VERSION = 1


def plan_header_bytes(N, c, I, itr, n_tasks):
    """Canonical plan header (format: include/cqs.h `cqs_plan_serialize`)."""
    b = PLAN_MAGIC + struct.pack("<I", PLAN_VERSION)
    b += struct.pack("<qii", N, c, len(I)) + struct.pack("<%di" % len(I), *I)
    b += struct.pack("<iq", itr, n_tasks)
    return b


def entry_bytes(entry: Entry) -> bytes:
    segs = entry_segments(entry)
    kept = segment_kept_matrix(entry, segs)
    b = struct.pack("<iQ", len(segs), entry_work(segs, kept))
    for (st, ln, cd) in segs:
        b += struct.pack("<qq", st, ln) + bytes(cd)
    for a in range(len(segs)):
        m = 0
        for bb in range(len(segs)):
            if kept[a, bb]:
                m |= 1 << bb
        b += struct.pack("<I", m)
    return b


def quorum_tuples_levels(cs):
    """All quorum tuples of a tree with c_t children at level t, lexicographic (R3)."""
    return list(itertools.product(*[range(c) for c in cs]))


def plan_bytes_levels(N, levels, itr) -> bytes:
    """Canonical bytes (version 3, include/cqs.h) of the uniform depth-`itr` tree whose level t
    uses levels[t] = (c_t, I_t) (R21), from the literal Algorithm 3 of every leaf."""
    b = PLAN_MAGIC + struct.pack("<I", 3) + struct.pack("<q", N) + struct.pack("<ii", itr, itr)
    for c, I in levels[:itr]:
        b += struct.pack("<ii", c, len(I)) + struct.pack("<%di" % len(I), *I)
    qts = quorum_tuples_levels([c for c, _ in levels[:itr]])
    b += struct.pack("<q", len(qts))
    for qt in qts:
        b += struct.pack("<i", itr) + entry_bytes(build_subseq_entry_levels(N, levels, qt))
    return b


def plan_bytes(N, c, I, itr) -> bytes:
    """Canonical bytes of the whole plan, from the literal Algorithm 3 (small/medium N)."""
    ents = build_subseq(N, c, itr, I)
    return plan_header_bytes(N, c, I, itr, len(ents)) + b"".join(entry_bytes(e) for e in ents)


def hybrid_plan_bytes(N, c, I, base_itr, leaves) -> bytes:
    """Canonical bytes of a hybrid plan (version 2, include/cqs.h): `leaves` = quorum paths of
    mixed length in DFS order; each leaf is the literal Algorithm 3 subsequence of its path."""
    b = PLAN_MAGIC + struct.pack("<I", 2)
    b += struct.pack("<qii", N, c, len(I)) + struct.pack("<%di" % len(I), *I)
    b += struct.pack("<iq", base_itr, len(leaves))
    for qt in leaves:
        b += struct.pack("<i", len(qt)) + entry_bytes(build_subseq_entry(N, c, I, tuple(qt)))
    return b


# ------------------------------------------------------------------------------------------------
# O7. Hybrid scheduling ("some subsequences at itr=1 can be further divided ... while others
#     remain unchanged"), DESIGN reading R20: which leaves to divide is this build's rule — start
#     from the uniform tree, LPT the leaves over `world` ranks, and while the makespan exceeds
#     1.01 x total/world divide the heaviest leaf (first in DFS order on ties) into its c children.
# ------------------------------------------------------------------------------------------------

def leaf_work(N, c, I, qt) -> int:
    e = build_subseq_entry(N, c, I, tuple(qt))
    segs = entry_segments(e)
    return entry_work(segs, segment_kept_matrix(e, segs))


def lpt(works, world):
    """LPT: largest first (stable on index), each to the least-loaded rank (lowest on ties).
    Returns (ranks, loads)."""
    order = sorted(range(len(works)), key=lambda i: -works[i])
    loads = [0] * world
    ranks = [-1] * len(works)
    for i in order:
        if works[i] == 0:
            continue
        r = min(range(world), key=lambda x: (loads[x], x))
        ranks[i] = r
        loads[r] += works[i]
    return ranks, loads


def hybrid_leaves(N, c, I, base_itr, world, tol=0.01, max_leaves=4096):
    leaves = [qt for qt in quorum_tuples(c, base_itr)]
    works = [leaf_work(N, c, I, qt) for qt in leaves]
    total = sum(works)
    while True:
        _, loads = lpt(works, world)
        if max(loads) <= (1 + tol) * total / world or len(leaves) + c - 1 > max_leaves:
            return leaves
        i = max(range(len(leaves)), key=lambda j: (works[j], -j))
        kids = [tuple(leaves[i]) + (q,) for q in range(c)]
        leaves[i:i + 1] = kids
        works[i:i + 1] = [leaf_work(N, c, I, qt) for qt in kids]


# ------------------------------------------------------------------------------------------------
# Coverage (Fig. 2 "all chunk pairs are covered exactly once")
# ------------------------------------------------------------------------------------------------

def coverage_counts(entries, N):
    """count[p, q] = number of entries in which global tokens p, q co-occur UNMASKED (brute force)."""
    cnt = np.zeros((N, N), dtype=np.int64)
    for e in entries:
        M = local_mask(e)
        ids = e.token_ids
        cnt[np.ix_(ids, ids)] += M.astype(np.int64)
    return cnt


# ------------------------------------------------------------------------------------------------
# O1. Dense softmax attention in float64 (the definition the method must reproduce, P:8)
# ------------------------------------------------------------------------------------------------

def dense_attention(q, k, v, alpha=None):
    """O = softmax(alpha Q K^T) V per (b, h) plane, row-max stabilised; also lse = log sum exp(alpha
    q.k).  q, k, v: float64 arrays [B, H, N, D].  Returns (O [B,H,N,D], lse [B,H,N])."""
    q = np.asarray(q, np.float64); k = np.asarray(k, np.float64); v = np.asarray(v, np.float64)
    D = q.shape[-1]
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    R = alpha * np.einsum("bhnd,bhmd->bhnm", q, k)
    m = R.max(axis=-1, keepdims=True)
    P = np.exp(R - m)
    s = P.sum(axis=-1, keepdims=True)
    O = np.einsum("bhnm,bhmd->bhnd", P, v) / s
    return O, (m + np.log(s))[..., 0]


def dense_attention_rows(q, k, v, rows, alpha=None, block=4096):
    """Same as dense_attention but only for query `rows` of one [N, D] plane, keys streamed in
    blocks: pass 1 takes the exact row max over all keys, pass 2 sums exp(logit - max) (the
    definition evaluated blockwise; no online rescaling).  q, k, v: [N, D] float64-convertible."""
    qr = np.asarray(q[rows], np.float64)
    N, D = k.shape
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    m = np.full(len(rows), -np.inf)
    for s in range(0, N, block):
        kb = np.asarray(k[s:s + block], np.float64)
        m = np.maximum(m, (alpha * qr @ kb.T).max(axis=1))
    den = np.zeros(len(rows)); num = np.zeros((len(rows), v.shape[1]))
    for s in range(0, N, block):
        kb = np.asarray(k[s:s + block], np.float64); vb = np.asarray(v[s:s + block], np.float64)
        P = np.exp(alpha * qr @ kb.T - m[:, None])
        den += P.sum(axis=1); num += P @ vb
    return num / den[:, None], m + np.log(den)


# ------------------------------------------------------------------------------------------------
# O3. Algorithm 1 literally: raw exp, Num/Den accumulators, IndexAdd
# ------------------------------------------------------------------------------------------------

def cqsa_forward_alg1(q, k, v, entries, alpha=None):
    """Algorithm 1 in float64 with the paper's raw exp (R7; valid while logits <
    709).  Returns O [B,H,N,D] and Den [B,H,N]."""
    B, H, N, D = q.shape
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    Num = np.zeros((B, H, N, D))
    Den = np.zeros((B, H, N))
    for e in entries:
        idx = e.token_ids
        Qi, Ki, Vi = q[:, :, idx], k[:, :, idx], v[:, :, idx]
        Mi = local_mask(e)
        Ri = alpha * np.einsum("bhld,bhmd->bhlm", Qi, Ki)
        assert Ri.max() < 700, "raw exp would overflow (R7)"
        Pi = np.exp(Ri) * Mi
        Numi = np.einsum("bhlm,bhmd->bhld", Pi, Vi)
        Deni = Pi.sum(axis=-1)
        np.add.at(Num, (slice(None), slice(None), idx), Numi)      # P:72 IndexAdd
        np.add.at(Den, (slice(None), slice(None), idx), Deni)
    return Num / Den[..., None], Den


# ------------------------------------------------------------------------------------------------
# O4. LSE form: per-task normalised partial (O_i, lse_i) and the LSE merge
# ------------------------------------------------------------------------------------------------

def task_partial(q, k, v, entry, alpha=None):
    """Per-task partial of Eq. 2 in the form an FA kernel returns:
    O_i = Num_i / Den_i, lse_i = log Den_i, computed with max stabilisation.  Rows with no kept key
    get O_i = 0, lse_i = -inf (R8)."""
    B, H, N, D = q.shape
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    idx = entry.token_ids
    Mi = local_mask(entry)
    Ri = alpha * np.einsum("bhld,bhmd->bhlm", q[:, :, idx], k[:, :, idx])
    Ri = np.where(Mi > 0, Ri, -np.inf)
    m = Ri.max(axis=-1, keepdims=True)
    msafe = np.where(np.isfinite(m), m, 0.0)
    Pi = np.exp(Ri - msafe)
    s = Pi.sum(axis=-1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        Oi = np.where(s > 0, np.einsum("bhlm,bhmd->bhld", Pi, v[:, :, idx]) / s, 0.0)
        lse = np.where(s[..., 0] > 0, (msafe + np.log(s))[..., 0], -np.inf)
    return Oi, lse


def lse_merge(parts):
    """Merge partials [(O_j, lse_j)] of the same rows (Eq. 3 with Den_j = exp(lse_j), Num_j =
    O_j Den_j): lse = log sum_j exp(lse_j); O = sum_j exp(lse_j - lse) O_j.
    -inf partials contribute nothing."""
    lses = np.stack([p[1] for p in parts])
    mx = lses.max(axis=0)
    msafe = np.where(np.isfinite(mx), mx, 0.0)
    w = np.exp(lses - msafe)
    tot = w.sum(axis=0)
    with np.errstate(divide="ignore"):
        lse = np.where(tot > 0, msafe + np.log(tot), -np.inf)
    O = sum(np.exp(p[1] - np.where(np.isfinite(lse), lse, 0.0))[..., None] * p[0] for p in parts)
    O = np.where(np.isfinite(lse)[..., None], O, 0.0)
    return O, lse


def cqsa_forward_lse(q, k, v, entries, alpha=None):
    """Algorithm 1 in LSE form: scatter each task's (O_i, lse_i) to global rows and LSE-merge all
    partials of a row (P:72-75 IndexAdd, P:240 reconstruction)."""
    B, H, N, D = q.shape
    parts = {n: [] for n in range(N)}
    for e in entries:
        Oi, li = task_partial(q, k, v, e, alpha)
        for loc, n in enumerate(e.token_ids):
            parts[int(n)].append((Oi[:, :, loc], li[:, :, loc]))
    O = np.zeros((B, H, N, D)); lse = np.zeros((B, H, N))
    for n in range(N):
        O[:, :, n], lse[:, :, n] = lse_merge(parts[n])
    return O, lse


# ------------------------------------------------------------------------------------------------
# O6. Backward: dense gradients and literal Algorithm 2
# ------------------------------------------------------------------------------------------------

def dense_attention_grads(q, k, v, dO, alpha=None):
    """Gradients of L = sum(dO * O), O = softmax(alpha Q K^T) V, per (b, h) plane, float64:
    dV = P^T dO;  dP = dO V^T;  dS = P * (dP - rowsum(dO * O));  dQ = alpha dS K;  dK = alpha dS^T Q.
    (The standard softmax chain rule; it is the Num/Den derivation of Appendix D collapsed with
    O = Num / Den.)"""
    q, k, v, dO = (np.asarray(t, np.float64) for t in (q, k, v, dO))
    D = q.shape[-1]
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    R = alpha * np.einsum("bhnd,bhmd->bhnm", q, k)
    P = np.exp(R - R.max(axis=-1, keepdims=True))
    P /= P.sum(axis=-1, keepdims=True)
    O = np.einsum("bhnm,bhmd->bhnd", P, v)
    dV = np.einsum("bhnm,bhnd->bhmd", P, dO)
    dP = np.einsum("bhnd,bhmd->bhnm", dO, v)
    delta = (dO * O).sum(axis=-1, keepdims=True)
    dS = P * (dP - delta)
    return alpha * np.einsum("bhnm,bhmd->bhnd", dS, k), alpha * np.einsum("bhnm,bhnd->bhmd", dS, q), dV


def cqsa_backward_alg2(q, k, v, dO, entries, alpha=None, only=None):
    """Algorithm 2 literally in float64, with Num / Den from Algorithm 1 (raw exp, R7):
    dNum = dO / Den; dDen = -rowsum(dO * Num) / Den^2 (Eq. 4); per task
    dV_i = P_i^T dNum_i; dP_i = dNum_i V_i^T + dDen_i 1^T; dR_i = dP_i * P_i; dQ_i = alpha dR_i K_i;
    dK_i = alpha dR_i^T Q_i (Eq. 5; dK uses Q_i, reading R18 for the P:484 typo);
    IndexAdd into dQ, dK, dV (Eq. 6).  `only` (optional set of task indices) restricts
    the loop of P:114 to those tasks — one rank's share of a task-sharded backward; the forward
    quantities Num / Den still come from all tasks."""
    q, k, v, dO = (np.asarray(t, np.float64) for t in (q, k, v, dO))
    B, H, N, D = q.shape
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    Num = np.zeros((B, H, N, D))
    Den = np.zeros((B, H, N))
    Ps = []
    for e in entries:                                              # forward (Alg. 1)
        idx = e.token_ids
        Pi = np.exp(alpha * np.einsum("bhld,bhmd->bhlm", q[:, :, idx], k[:, :, idx])) * local_mask(e)
        Ps.append(Pi)
        np.add.at(Num, (slice(None), slice(None), idx), np.einsum("bhlm,bhmd->bhld", Pi, v[:, :, idx]))
        np.add.at(Den, (slice(None), slice(None), idx), Pi.sum(axis=-1))
    dQ, dK, dV = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    dNum = dO / Den[..., None]
    dDen = -(dO * Num).sum(axis=-1) / (Den * Den)
    for t, (e, Pi) in enumerate(zip(entries, Ps)):
        if only is not None and t not in only:
            continue
        idx = e.token_ids
        dNum_i, dDen_i = dNum[:, :, idx], dDen[:, :, idx]
        dV_i = np.einsum("bhlm,bhld->bhmd", Pi, dNum_i)
        dP_i = np.einsum("bhld,bhmd->bhlm", dNum_i, v[:, :, idx]) + dDen_i[..., None]
        dR_i = dP_i * Pi
        dQ_i = alpha * np.einsum("bhlm,bhmd->bhld", dR_i, k[:, :, idx])
        dK_i = alpha * np.einsum("bhlm,bhld->bhmd", dR_i, q[:, :, idx])
        np.add.at(dQ, (slice(None), slice(None), idx), dQ_i)
        np.add.at(dK, (slice(None), slice(None), idx), dK_i)
        np.add.at(dV, (slice(None), slice(None), idx), dV_i)
    return dQ, dK, dV


def dense_dq_rows(q, k, v, dO, rows, alpha=None, block=1 << 16):
    """dQ for query `rows` of one [N, D] plane (the dQ of dense_attention_grads row by row, for
    sizes where the full N x N matrices do not fit): O_r and lse_r from dense_attention_rows, then
    dQ_r = alpha sum_j P_rj (dO_r . v_j - dO_r . O_r) k_j with keys streamed in blocks."""
    N, D = k.shape
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    Or, lse = dense_attention_rows(q, k, v, rows, alpha, block)
    qr = np.asarray(q[rows], np.float64)
    dOr = np.asarray(dO[rows], np.float64)
    delta = (dOr * Or).sum(axis=1)
    dq = np.zeros((len(rows), D))
    for s in range(0, N, block):
        kb = np.asarray(k[s:s + block], np.float64); vb = np.asarray(v[s:s + block], np.float64)
        P = np.exp(alpha * qr @ kb.T - lse[:, None])
        dq += (P * (dOr @ vb.T - delta[:, None])) @ kb
    return alpha * dq
