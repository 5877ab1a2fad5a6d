"""CPU oracle of the EPS-MoE MoE-layer hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  It shares no code with the
CUDA path (``paper_2410_12247_b200/``) and never imports it.

Citations: ``P:n`` = line n of the paper's LaTeX (arXiv 2410.12247, PAPER.md);
readings ``R1..R17`` are listed in DESIGN.md §3.

EPS-MoE is an exact *schedule* (P:221-222): it computes the plain MoE
layer

    y_t = FFN_shared(x_t) + sum_{j<k} w_{t,j} * FFN_{e_{t,j}}(x_t),
    FFN_e(x) = (silu(x W_gate,e^T) * (x W_up,e^T)) W_down,e^T

faster.  The oracle is therefore that definition, executed as the paper's
Algorithm 1 over D simulated ranks and PN chunks, so that the
integer artefacts (histograms, counts, offsets, permutation) are defined too:

    index <- Router(input)                       router_logits + topk_gating
    m <- count(input) ; tensor[] <- split(...)   dispatch_layout
    All2All / ComputeMoE / All2All per chunk     expert_ffn on each chunk's rows
    LocalReduce (home-side weighted sum, R7)     combine
    or expert-side LocalReduce + dedup (R16)     lr_layout, local_reduce_combine

Two numeric modes (R4):
  * "exact":    fp64 everywhere, no intermediate rounding;
  * "contract": fp64 accumulation, rounded to fp32 / bf16 at exactly the GPU's
                points: logits fp32; g,u fp32; h bf16; o bf16; s bf16;
                combine = fp32 fmaf chain from s in slot order; y bf16.
Library primitives used as steps: numpy matmul (fp64) and exp.

Pins (tests/test_oracle_pins.py): brute force per token, dense-MLP special case
vs torch fp64, exact-logit grid, tie fixture, k=E, activated-experts formula
(P:133), the fig:eps_overview worked example, conservation,
chunked == unchunked, EP=D == EP=1; FP8 codec vs the e4m3 format definition;
LocalReduce (R16): the worked example's dedup counts by hand, exact-mode
regrouping identity, single-group special case, the hypergeometric
distinct-rank closed form; device-limited routing (R17): a hand fixture, the
M = groups special case; the P:265 all2all volume bounds; chunk groups vs the
SURVEY §8(c) table, token slices / shards / sliced send counts vs hand tables
(tests/golden/chunk_rules.json); the contract combine vs an exact-rational
fmaf chain with crafted tokens that expose s-last and mul+add.
"""
from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# rounding helpers (R4).  Plain bit manipulation, round-to-nearest-even.
# ----------------------------------------------------------------------------


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def round_bf16(v) -> np.ndarray:
    """fp32 value(s) -> nearest-even bf16 value, returned as float32."""
    f = np.asarray(v, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    r = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def bf16_value_to_bits(v: np.ndarray) -> np.ndarray:
    return (np.asarray(v, dtype=np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def fmaf(a: np.ndarray, b: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Correctly rounded fp32 a*b+c for fp32 a, c and b with <= 24 significant bits.

    a*b is exact in fp64 (<= 48 significant bits).  s = fl64(p + c) may carry a
    rounding error e (recovered exactly by TwoSum); the final fp32 rounding of s
    is then correct unless s sits exactly on an fp32 rounding midpoint, in which
    case the sign of e decides (double-rounding guard).
    """
    a = np.asarray(a, np.float32).astype(np.float64)
    b = np.asarray(b, np.float32).astype(np.float64)
    c = np.asarray(c, np.float32).astype(np.float64)
    p = a * b
    s = p + c
    bb = s - p
    e = (p - (s - bb)) + (c - bb)              # TwoSum: p + c == s + e exactly
    bits = s.view(np.uint64)
    mid = (bits & np.uint64((1 << 29) - 1)) == np.uint64(1 << 28)
    fix = mid & (e != 0)
    if np.any(fix):
        s = s.copy()
        s[fix] = np.nextafter(s[fix], np.where(e[fix] > 0, np.inf, -np.inf))
    return s.astype(np.float32)


def silu_f32(g: np.ndarray) -> np.ndarray:
    """silu(g) = g / (1 + e^-g) evaluated in fp32 (R4)."""
    g = np.asarray(g, np.float32)
    with np.errstate(over="ignore"):
        return (g / (np.float32(1.0) + np.exp(-g))).astype(np.float32)


# ----------------------------------------------------------------------------
# FP8 dispatch payload (Table II "FP8" column P:312/331; NEXT-2, R15).
# ----------------------------------------------------------------------------

E4M3_MAX = 448.0
FP8_BLOCK = 128


def fp8_block_exponent(amax: float) -> int:
    """Smallest s with amax / 2^s <= 448 (power-of-two block scale, R15).
    amax = m 2^e with 1 <= m < 2 and 448 = 1.75 2^8, so s = e-8 if m <= 1.75
    else e-7; clamped to s >= -126 (2^s a normal fp32).  amax == 0 -> -126."""
    if amax == 0.0:
        return -126
    m, e = np.frexp(np.float64(amax))       # amax = m 2^e, 0.5 <= m < 1
    m, e = 2.0 * m, int(e) - 1               # 1 <= m < 2
    return max(-126, e - 8 if m <= 1.75 else e - 7)


def fp8_dispatch_roundtrip(x_bits: np.ndarray) -> np.ndarray:
    """The value an expert receives for a row dispatched in FP8 (R15):
    per 128-column block, s = fp8_block_exponent(max|x|), q = e4m3_rne(x 2^-s)
    (never saturates: |x 2^-s| <= 448), x' = q 2^s (exact in bf16).
    Returns bf16 bit patterns.  e4m3 rounding uses torch's float8_e4m3fn cast
    (a library routine; RNE)."""
    import torch
    x = bf16_bits_to_f64(x_bits)
    out = np.empty_like(x)
    rows, cols = x.shape
    for b0 in range(0, cols, FP8_BLOCK):
        blk = x[:, b0:b0 + FP8_BLOCK]
        for r in range(rows):
            s = fp8_block_exponent(float(np.abs(blk[r]).max()))
            v = blk[r] * np.float64(2.0) ** (-s)                 # exact (power of two)
            q = torch.from_numpy(v.astype(np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()
            out[r, b0:b0 + FP8_BLOCK] = q * np.float64(2.0) ** s
    return bf16_value_to_bits(out.astype(np.float32))


# ----------------------------------------------------------------------------
# Step 1: Router (Alg. 1 line `index <- Router(input)`).
# ----------------------------------------------------------------------------


def router_logits(x_bits, w_router_bits, router_bias=None, mode="contract"):
    """logits[t,e] = sum_h x[t,h] W_r[e,h] (+ beta_e, the synthetic skew hook).

    contract: fp32(fp64 sum), then one fp32 add of beta (R1).
    """
    x = bf16_bits_to_f64(x_bits)
    w = bf16_bits_to_f64(w_router_bits)
    l64 = x @ w.T
    if mode == "exact":
        if router_bias is not None:
            l64 = l64 + np.asarray(router_bias, np.float64)[None, :]
        return l64
    l32 = l64.astype(np.float32)
    if router_bias is not None:
        l32 = (l32 + np.asarray(router_bias, np.float32)[None, :]).astype(np.float32)
    return l32


# ----------------------------------------------------------------------------
# Step 2: topKGating.  Readings R1 (softmax over all E, select on
# logits, norm_topk for Mixtral), R2 (ties -> lower expert id).
# ----------------------------------------------------------------------------


def topk_gating(logits, k, norm_topk, routed_scale=1.0, mode="contract", route_groups=0, route_topk_groups=0):
    """Returns (idx [T,k] int32, w [T,k] float32; float64 in exact mode).

    idx_t = the k experts ordered by (logit desc, expert id asc).
    p = softmax over all E (computed in fp64 from the fp32 logits, rounded to
    fp32); w_j = p_{idx_j}; if norm_topk: w_j = p_{idx_j} / sum_j p_{idx_j};
    then w_j *= routed_scale.

    Device-limited routing (DeepSeek-V2's mechanism; NEXT-4, R17) when
    1 < route_groups and route_topk_groups < route_groups: the E experts form
    route_groups contiguous groups of E/route_groups; a group's score is its
    largest logit; only the experts of the route_topk_groups best groups
    (score desc, group id asc) are eligible for the top-k above.  The softmax
    still runs over all E.

    A NaN logit (from NaN / Inf inputs only) ranks as -inf: never selected
    ahead of a number, 0 in the softmax (R18).  A row of NaNs selects experts
    0..k-1 and gets NaN weights (its max is -inf).
    """
    logits = np.asarray(logits)
    T, E = logits.shape
    idx = np.empty((T, k), dtype=np.int32)
    w = np.empty((T, k), dtype=np.float64 if mode == "exact" else np.float32)
    experts = np.arange(E)
    limited = route_groups > 1 and route_topk_groups < route_groups
    if limited:
        gsz = E // route_groups
        groups = np.arange(route_groups)
    for t in range(T):
        row = logits[t].astype(np.float64)
        row = np.where(np.isnan(row), -np.inf, row)  # a NaN logit ranks as -inf (R18)
        order = np.lexsort((experts, -row))          # primary: -logit, secondary: e
        if limited:
            score = row.reshape(route_groups, gsz).max(axis=1)
            keep = np.lexsort((groups, -score))[:route_topk_groups]
            order = order[np.isin(order // gsz, keep)]
        sel = order[:k]
        ex = np.exp(row - row.max())
        p = ex / ex.sum()
        ps = p[sel]
        if norm_topk:
            ps = ps / ps.sum()
        idx[t] = sel
        w[t] = ps * routed_scale
    return idx, w


# ----------------------------------------------------------------------------
# Step 3: count + split + the all2all layouts (Alg. 1; R6, R8, R12).
# ----------------------------------------------------------------------------


def token_shards(T, D):
    """Rank r owns global tokens [start[r], start[r+1]); first T mod D get +1 (R12)."""
    base, rem = divmod(T, D)
    sizes = [base + (1 if r < rem else 0) for r in range(D)]
    start = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return start


def chunk_groups(E_loc, N):
    """Balanced contiguous groups of local experts (R8): the first
    E_loc mod N groups get ceil(E_loc/N) experts.  Returns begin[N+1]."""
    if not (1 <= N <= E_loc):
        raise ValueError("need 1 <= N <= E_loc")
    base, rem = divmod(E_loc, N)
    sizes = [base + (1 if c < rem else 0) for c in range(N)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def slice_ranges(T_loc, S):
    """Balanced contiguous source-token ranges for token_slices S (R8 extension)."""
    base, rem = divmod(T_loc, S)
    sizes = [base + (1 if s < rem else 0) for s in range(S)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def dispatch_layout(idx, E, D):
    """Per-rank integer artefacts of `split` and the all2all layouts.

    Send buffer on rank r: the rank's (t, j) pairs ordered by (e asc, t asc)
    (R6).  Recv buffer on rank d: rows ordered by (local expert asc, src asc,
    t asc).  Both orders are chunk-independent; chunk c = the contiguous
    sub-ranges of its experts (R8).

    Returns dict with, per rank r:
      hist[r][e]          pairs of rank r routed to expert e
      pos[r] [T_loc,k]    send row of pair (t, j)
      send_start[r][e]    first send row of expert e on rank r
      recv_start[d][e_l][src]  first recv row of (local expert e_l, src) on d
      recv_total[d]       rows received by d
    """
    T, k = idx.shape
    E_loc = E // D
    start = token_shards(T, D)
    hist = np.zeros((D, E), dtype=np.int64)
    pos = []
    send_start = np.zeros((D, E + 1), dtype=np.int64)
    for r in range(D):
        loc = idx[start[r]:start[r + 1]]
        for e in range(E):
            hist[r, e] = int(np.count_nonzero(loc == e))
        send_start[r, 1:] = np.cumsum(hist[r])
        p = np.full(loc.shape, -1, dtype=np.int64)
        nxt = send_start[r, :E].copy()
        for t in range(loc.shape[0]):          # token order => stable within e
            for j in range(k):
                e = loc[t, j]
                p[t, j] = nxt[e]
                nxt[e] += 1
        pos.append(p)
    recv_start = np.zeros((D, E_loc, D), dtype=np.int64)
    recv_total = np.zeros(D, dtype=np.int64)
    for d in range(D):
        row = 0
        for el in range(E_loc):
            e = d * E_loc + el
            for src in range(D):
                recv_start[d, el, src] = row
                row += hist[src, e]
        recv_total[d] = row
    return dict(hist=hist, pos=pos, send_start=send_start, recv_start=recv_start,
                recv_total=recv_total, token_start=start)


def chunk_send_counts(hist, E, D, N, token_slices=1, idx=None):
    """send[c][src][dst] = rows src sends dst in chunk c (all2all dispatch sizes).

    Chunk id c = group * token_slices + slice (R8).  With token_slices > 1 the
    per-slice counts need the routing itself (idx)."""
    E_loc = E // D
    gb = chunk_groups(E_loc, N)
    C = N * token_slices
    send = np.zeros((C, D, D), dtype=np.int64)
    if token_slices == 1:
        for g in range(N):
            for src in range(D):
                for dst in range(D):
                    es = range(dst * E_loc + gb[g], dst * E_loc + gb[g + 1])
                    send[g, src, dst] = sum(int(hist[src, e]) for e in es)
        return send
    start = token_shards(idx.shape[0], D)
    for src in range(D):
        loc = idx[start[src]:start[src + 1]]
        sr = slice_ranges(loc.shape[0], token_slices)
        for g in range(N):
            for s in range(token_slices):
                part = loc[sr[s]:sr[s + 1]]
                for dst in range(D):
                    lo, hi = dst * E_loc + gb[g], dst * E_loc + gb[g + 1]
                    send[g * token_slices + s, src, dst] = int(np.count_nonzero((part >= lo) & (part < hi)))
    return send


# ----------------------------------------------------------------------------
# Step 4: ComputeMoE: GateUpGemm -> SiluAct -> DownGemm.
# ----------------------------------------------------------------------------


def expert_ffn(a_bits, wg_bits, wu_bits, wd_bits, mode="contract"):
    """SwiGLU expert on rows A [n,H] (bf16 bits).  Returns o [n,H]:
    contract -> float32 holding bf16 values; exact -> float64."""
    A = bf16_bits_to_f64(a_bits)
    Wg = bf16_bits_to_f64(wg_bits)
    Wu = bf16_bits_to_f64(wu_bits)
    Wd = bf16_bits_to_f64(wd_bits)
    g = A @ Wg.T                                   # GateUpGemm
    u = A @ Wu.T
    if mode == "exact":
        h = g / (1.0 + np.exp(-g)) * u             # SiluAct
        return h @ Wd.T                            # DownGemm
    g32 = g.astype(np.float32)
    u32 = u.astype(np.float32)
    h = round_bf16((silu_f32(g32) * u32).astype(np.float32))      # h -> bf16
    o32 = (h.astype(np.float64) @ Wd.T).astype(np.float32)
    return round_bf16(o32)                                         # o -> bf16


# ----------------------------------------------------------------------------
# Step 5: LocalReduce / combine (R7, R10).
# ----------------------------------------------------------------------------


def combine(s, o_slots, w, mode="contract"):
    """y_t = s_t + sum_j w_j o_{t,j}.  contract: acc = fp32(s); for j in slot
    order acc = fmaf(w_j, o_j, acc); y = bf16(acc).  o_slots: [T,k,H]."""
    T, k, H = o_slots.shape
    if mode == "exact":
        y = np.array(s, dtype=np.float64, copy=True)
        for j in range(k):
            y = y + w[:, j].astype(np.float64)[:, None] * o_slots[:, j, :]
        return y
    acc = np.asarray(s, np.float32).copy()
    for j in range(k):
        acc = fmaf(np.broadcast_to(w[:, j][:, None], (T, H)), o_slots[:, j, :], acc)
    return round_bf16(acc)


# ----------------------------------------------------------------------------
# NEXT-3 / R16: expert-side LocalReduce with per-(token, destination, chunk)
# dedup.  ComputeMoE ends with LocalReduce(tensor) on the expert side
# (P:559); fig:comp_overlap_comm and P:365 place it before the second
# all2all, which it overlaps.  So each token travels once per (destination
# rank, chunk) and returns as one partial sum of its experts there.
# ----------------------------------------------------------------------------


def lr_group_ids(idx, E, D, N):
    """Group of pair (t, j): g = c * D + d, with d = e // E_loc the rank owning
    e = idx[t, j] (EP) and c the chunk holding e's local id e % E_loc
    (balanced contiguous groups of local experts, R8)."""
    E_loc = E // D
    gb = chunk_groups(E_loc, N)
    chunk_of = np.searchsorted(gb, np.arange(E_loc), side="right") - 1
    idx = np.asarray(idx, np.int64)
    return chunk_of[idx % E_loc] * D + idx // E_loc


def lr_layout(idx, E, D, N):
    """Dedup all2all layout (R16), per rank r of the token shards (R12):

      gid[r]     [T_loc, k]  group of each pair (lr_group_ids)
      u_hist[r]  [G]         rows r sends for group g = c*D + d: the distinct
                             tokens of r with a pair in g (to rank d, chunk c)
      u_start[r] [G+1]       send rows ordered by (g asc, t asc)
      posg[r]    [T_loc, k]  send row of t's i-th distinct group (groups in
                             ascending g), -1 past the token's group count
      recv_u_start[d] [N, D] first row, in d's receive buffer ordered by
                             (c asc, src asc, t asc), of what src sends d in c
    G = N * D."""
    T, k = idx.shape
    E_loc = E // D
    G = N * D
    start = token_shards(T, D)
    gid_all = lr_group_ids(idx, E, D, N)
    gid, u_hist, u_start, posg = [], np.zeros((D, G), np.int64), np.zeros((D, G + 1), np.int64), []
    for r in range(D):
        gr = gid_all[start[r]:start[r + 1]]
        T_loc = gr.shape[0]
        for g in range(G):
            u_hist[r, g] = int(np.count_nonzero((gr == g).any(axis=1)))
        u_start[r, 1:] = np.cumsum(u_hist[r])
        nxt = u_start[r, :G].copy()
        pg = np.full((T_loc, k), -1, np.int64)
        for t in range(T_loc):                 # token order => stable within g
            for i, g in enumerate(sorted(set(int(v) for v in gr[t]))):
                pg[t, i] = nxt[g]
                nxt[g] += 1
        gid.append(gr)
        posg.append(pg)
    recv_u_start = np.zeros((D, N, D), np.int64)
    for d in range(D):
        row = 0
        for c in range(N):
            for src in range(D):
                recv_u_start[d, c, src] = row
                row += u_hist[src, c * D + d]
    return dict(gid=gid, u_hist=u_hist, u_start=u_start, posg=posg, recv_u_start=recv_u_start,
                token_start=start, E_loc=E_loc)


def local_reduce_combine(s, o_slots, w, gid, mode="contract"):
    """y under R16.  Expert side, per distinct group g of token t:
        acc = 0; for j ascending with gid[t, j] == g: acc = fmaf(w_j, o_{t,j}, acc);
        p_{t,g} = bf16(acc)                                (LocalReduce)
    home side, after all2all_combine:
        acc = fp32(s_t); for g ascending: acc = acc + p_{t,g}; y_t = bf16(acc).
    exact: y = s + sum_g sum_{j in g} w_j o_j in fp64.  o_slots: [T,k,H]."""
    T, k, H = o_slots.shape
    gid = np.asarray(gid, np.int64)
    gs = np.sort(gid, axis=1)
    distinct = np.ones_like(gs, dtype=bool)
    distinct[:, 1:] = gs[:, 1:] != gs[:, :-1]
    if mode == "exact":
        y = np.array(s, dtype=np.float64, copy=True)
        for i in range(k):
            for t in np.nonzero(distinct[:, i])[0]:
                part = np.zeros(H)
                for j in range(k):
                    if gid[t, j] == gs[t, i]:
                        part = part + float(w[t, j]) * o_slots[t, j]
                y[t] = y[t] + part
        return y
    acc = np.asarray(s, np.float32).copy()
    for i in range(k):                      # i-th slot of the sorted group list
        rows = np.nonzero(distinct[:, i])[0]
        if rows.size == 0:
            continue
        g = gs[rows, i]
        part = np.zeros((rows.size, H), np.float32)
        for j in range(k):                  # slot order inside the group
            m = gid[rows, j] == g
            if m.any():
                rj = rows[m]
                part[m] = fmaf(np.broadcast_to(np.asarray(w, np.float32)[rj, j][:, None], (rj.size, H)),
                               o_slots[rj, j, :], part[m])
        p = round_bf16(part)                # the combine payload is bf16
        acc[rows] = (acc[rows] + p).astype(np.float32)
    return round_bf16(acc)


# ----------------------------------------------------------------------------
# The layer (Algorithm 1), simulated over D ranks and PN chunks.
# ----------------------------------------------------------------------------


def moe_layer(x_bits, w_router_bits, w_gate_bits, w_up_bits, w_down_bits, k, norm_topk,
              ws_gate_bits=None, ws_up_bits=None, ws_down_bits=None, router_bias=None,
              routed_scale=1.0, D=1, N=1, token_slices=1, mode="contract",
              topk_override=None, dispatch_fp8=False, local_reduce=False, route_groups=0,
              route_topk_groups=0):
    """Full layer over all T tokens.  Weights are indexed by global expert id.

    topk_override = (idx, w) replaces Router + topKGating (explicit routing,
    used by the fig:eps_overview fixture).  dispatch_fp8: every dispatched row
    travels as FP8 (fp8_dispatch_roundtrip, R15); shared experts see x.
    local_reduce: expert-side LocalReduce with per-(token, destination,
    chunk) dedup (R16): the rows each expert sees are unchanged, only the sum
    is regrouped (local_reduce_combine); the result adds the dedup layout.
    """
    T, H = x_bits.shape
    E = w_gate_bits.shape[0]
    if E % D:
        raise ValueError("E % D != 0 is rejected (R12)")
    E_loc = E // D
    if topk_override is None:
        logits = router_logits(x_bits, w_router_bits, router_bias, mode)
        idx, w = topk_gating(logits, k, norm_topk, routed_scale, mode, route_groups, route_topk_groups)
    else:
        logits = None
        idx, w = (np.asarray(a) for a in topk_override)
        idx = idx.astype(np.int32)
        w = w.astype(np.float64 if mode == "exact" else np.float32)
    lay = dispatch_layout(idx, E, D)
    start = lay["token_start"]
    gb = chunk_groups(E_loc, N)

    # Send buffers (split): row pos[r][t,j] of rank r holds x[t]
    # (or its FP8 round trip when the dispatch payload is FP8).
    x_disp = fp8_dispatch_roundtrip(x_bits) if dispatch_fp8 else x_bits
    send = []
    for r in range(D):
        buf = np.zeros((int(lay["send_start"][r, E]), H), dtype=np.uint16)
        p = lay["pos"][r]
        for t in range(p.shape[0]):
            for j in range(k):
                buf[p[t, j]] = x_disp[start[r] + t]
        send.append(buf)

    # Dispatch -> ComputeMoE -> combine, chunk by chunk.  The
    # result rows land back in each home rank's combine buffer at the send row.
    comb = [np.zeros((b.shape[0], H), dtype=np.float64 if mode == "exact" else np.float32)
            for b in send]
    for g in range(N):
        for sl in range(token_slices):
            for d in range(D):                       # expert owner
                for el in range(gb[g], gb[g + 1]):
                    e = d * E_loc + el
                    for src in range(D):
                        # rows of (e, src) in this token slice, in src token order
                        T_loc = int(start[src + 1] - start[src])
                        sr = slice_ranges(T_loc, token_slices)
                        loc = idx[start[src]:start[src + 1]]
                        tok, slot = np.nonzero(loc == e)
                        keep = (tok >= sr[sl]) & (tok < sr[sl + 1])
                        tok, slot = tok[keep], slot[keep]
                        if tok.size == 0:
                            continue
                        rows = lay["pos"][src][tok, slot]
                        a = send[src][rows]                       # All2All dispatch
                        o = expert_ffn(a, w_gate_bits[e], w_up_bits[e], w_down_bits[e], mode)
                        comb[src][rows] = o                       # All2All combine

    # Shared experts (R10): one MLP of width S*F_s on the home rank.
    if ws_gate_bits is not None:
        s = expert_ffn(x_bits, ws_gate_bits, ws_up_bits, ws_down_bits, mode)
    else:
        s = np.zeros((T, H), dtype=np.float64 if mode == "exact" else np.float32)

    o_slots = np.zeros((T, k, H), dtype=comb[0].dtype if comb else np.float32)
    for r in range(D):
        p = lay["pos"][r]
        o_slots[start[r]:start[r + 1]] = comb[r][p]
    out = dict(logits=logits, idx=idx, w=w, s=s, layout=lay,
               send_counts=chunk_send_counts(lay["hist"], E, D, N, token_slices, idx), group_begin=gb)
    if local_reduce:
        if token_slices != 1:
            raise ValueError("local_reduce: token_slices must be 1")
        lr = lr_layout(idx, E, D, N)
        out["lr_layout"] = lr
        out["y"] = local_reduce_combine(s, o_slots, w, np.concatenate(lr["gid"]), mode)
    else:
        out["y"] = combine(s, o_slots, w, mode)
    return out


def moe_tokens(x_bits, w_router_bits, expert_weights, k, norm_topk, shared=None,
               router_bias=None, routed_scale=1.0, mode="contract", dispatch_fp8=False, route_groups=0,
               route_topk_groups=0):
    """y for an arbitrary subset of tokens (y_t depends only on x_t and the
    weights).  expert_weights: callable e -> (Wg, Wu, Wd) bits.
    Used for sampled parity at the full BASELINE sizes."""
    logits = router_logits(x_bits, w_router_bits, router_bias, mode)
    idx, w = topk_gating(logits, k, norm_topk, routed_scale, mode, route_groups, route_topk_groups)
    T, H = x_bits.shape
    x_disp = fp8_dispatch_roundtrip(x_bits) if dispatch_fp8 else x_bits
    o_slots = np.zeros((T, k, H), dtype=np.float64 if mode == "exact" else np.float32)
    for e in np.unique(idx):
        tok, slot = np.nonzero(idx == e)
        wg, wu, wd = expert_weights(int(e))
        o_slots[tok, slot] = expert_ffn(x_disp[tok], wg, wu, wd, mode)
    if shared is not None:
        s = expert_ffn(x_bits, *shared, mode)
    else:
        s = np.zeros((T, H), dtype=o_slots.dtype)
    y = combine(s, o_slots, w, mode)
    return dict(logits=logits, idx=idx, w=w, y=y)
