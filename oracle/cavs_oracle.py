"""CPU oracle for Cavs' level-batched F-over-G hot path.  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import or call this module.  It shares no code
with the CUDA path (`paper_1712_04048_b200/`); its only common inputs are the
arrays drawn by `workloads/`.

What it computes (PAPER.md = /root/reference/PAPER.md, "P:Lnnn" = line):
  * validation of the input graphs G (SPEC S:L166 arity),
    cycle detection by three-colour DFS;
  * the schedule of Algorithm 1, two independent ways:
    (i) level(v) = 0 for a vertex without children, else 1 + max over its
        children (the "activated iff all dependent vertices evaluated" rule,
        P:L357, read as SURVEY Z5), by memoised recursion;
    (ii) a literal simulation of Alg. 1's FORWARD loop;
    order inside a task V_t = ascending global vertex id (reading Z4);
  * the forward pass as the plain definition: a per-vertex recursive
    evaluator that evaluates all children first, then applies F (Fig. 5,
    P:L314-331 for the N-ary child-sum Tree-LSTM; Tree-FC per reading Z7:
    h = tanh(W_l h_l + W_r h_r + W_x x + b), "a single fully-connected layer",
    P:L608; LSTM = Tree-LSTM with N = 1);
  * missing children and absent pull records are zero vectors (reading Z1/Z2);
  * the loss is external: L = sum_v <Gamma_v, h_v>, so dL/dh_push = Gamma;
  * the backward pass in exactly the reverse of the forward evaluation order
    (P:L358), gradients ADDED, never overwritten;
    gather's adjoint is scatter and pull's adjoint is push.
  * fp64 throughout (the paper never states a precision, Z11).  The optional
    `emulate_bf16=True` mode is a DIAGNOSTIC (it separates bf16 quantisation
    from bugs; the parity gate is always the plain fp64 mode): it rounds the
    GEMM operands of SURVEY reading Z11 (params W,U; x; the gathered h_k and
    the child-sum h~; the stored dZ) RN-even via fp32 (pin P9).  Fig. 5 fixes
    U h~ with h~ = sum_k h_k but no rounding point, so two bf16 readings are
    offered:
      bf16_hsum="rounded" (default, Z11 as written): h~ = bf16(sum_k bf16(h_k));
      bf16_hsum="exact"   (reading R-lin): U h~ taken as sum_k U bf16(h_k) in
                          exact arithmetic, i.e. h~ = sum_k bf16(h_k) unrounded.
    Both equal the fp64 definition up to bf16 rounding; they coincide bit for
    bit when no vertex has two or more children.
  * `accum="fp32"` (diagnostic, any mode) evaluates the matrix-vector products
    in fp32 instead of fp64: a second valid evaluation, whose distance from the
    fp64 one measures how much a chaotic F (reading R-chaos) amplifies rounding
    -- the conditioning-derived parity band of the cfg5 bench init.

Parity status: every function here is pinned by `tests/test_oracle_pins.py`
(closed forms, brute force, torch.nn.LSTM, finite differences, hand-worked
examples tests/golden/*.json).  The Tree-FC *cell form* itself is a reading
(Z7) the paper does not fix; its arithmetic is pinned by W3/W4 and FD.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np

TREE_LSTM = "tree_lstm"
TREE_FC = "tree_fc"


class OracleError(Exception):
    """Validation failure; `code` in {"invalid", "arity", "cycle", "fanout"}."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


# ---------------------------------------------------------------------------
# precision helpers
# ---------------------------------------------------------------------------
def f32(a):
    """Round to fp32 (the GPU holds every state value in fp32)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def bf16r(a):
    """Round to bf16, RN-even, via fp32 (what __float2bfloat16_rn does to an fp32 value)."""
    u = np.asarray(a, dtype=np.float32).copy().view(np.uint32)
    u = (u + (np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1)))) & np.uint32(0xFFFF0000)
    return u.view(np.float32).astype(np.float64)


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------
def global_children(graph_ptr, child_ptr, child_idx):
    """children[v] as GLOBAL ids: global id = graph_ptr[k] + local id."""
    K = len(graph_ptr) - 1
    V = int(graph_ptr[-1])
    ch = []
    for k in range(K):
        base = int(graph_ptr[k])
        for v in range(base, int(graph_ptr[k + 1])):
            ch.append([base + int(c) for c in child_idx[child_ptr[v]:child_ptr[v + 1]]])
    assert len(ch) == V
    return ch


def validate(graph_ptr, child_ptr, child_idx, N, allow_fanout=True):
    """Checks of the input-graph contract; raises OracleError."""
    K = len(graph_ptr) - 1
    if K < 1:
        raise OracleError("invalid", "K >= 1 graphs required")
    V = int(graph_ptr[-1])
    if int(graph_ptr[0]) != 0 or len(child_ptr) != V + 1:
        raise OracleError("invalid", "graph_ptr/child_ptr shape")
    for k in range(K):
        if graph_ptr[k + 1] - graph_ptr[k] < 1:
            raise OracleError("invalid", f"graph {k} is empty")
    n_parents = np.zeros(V, dtype=np.int64)
    for k in range(K):
        nk = int(graph_ptr[k + 1] - graph_ptr[k])
        for v in range(int(graph_ptr[k]), int(graph_ptr[k + 1])):
            deg = int(child_ptr[v + 1] - child_ptr[v])
            if deg < 0:
                raise OracleError("invalid", "child_ptr not monotone")
            if deg > N:
                raise OracleError("arity", f"vertex {v} has {deg} > N={N} children")
            for c in child_idx[child_ptr[v]:child_ptr[v + 1]]:
                if not (0 <= int(c) < nk):
                    raise OracleError("invalid", f"child id {int(c)} out of range in graph {k}")
                n_parents[int(graph_ptr[k]) + int(c)] += 1
    ch = global_children(graph_ptr, child_ptr, child_idx)
    # three-colour DFS (iterative) for cycles
    colour = np.zeros(V, dtype=np.int8)  # 0 white, 1 grey, 2 black
    for s in range(V):
        if colour[s]:
            continue
        stack = [(s, 0)]
        colour[s] = 1
        while stack:
            v, i = stack[-1]
            if i < len(ch[v]):
                stack[-1] = (v, i + 1)
                c = ch[v][i]
                if colour[c] == 1:
                    raise OracleError("cycle", f"cycle through vertex {c}")
                if colour[c] == 0:
                    colour[c] = 1
                    stack.append((c, 0))
            else:
                colour[v] = 2
                stack.pop()
    if not allow_fanout and np.any(n_parents > 1):
        raise OracleError("fanout", "a vertex has more than one parent")
    return ch


def levels_recursive(children):
    """level(v) = 0 if v has no children else 1 + max_k level(child_k) (Z5)."""
    V = len(children)
    level = [-1] * V
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 4 * V + 1000))

    def lev(v):
        if level[v] < 0:
            level[v] = 0 if not children[v] else 1 + max(lev(c) for c in children[v])
        return level[v]

    try:
        for v in range(V):
            lev(v)
    finally:
        sys.setrecursionlimit(old)
    return np.asarray(level, dtype=np.int32)


def schedule_alg1(children):
    """Literal Algorithm 1 FORWARD: repeatedly take ALL activated
    vertices (not evaluated, every child evaluated) as V_t, push, mark evaluated."""
    V = len(children)
    evaluated = [False] * V
    S = []
    n_done = 0
    while n_done < V:
        Vt = [v for v in range(V)
              if not evaluated[v] and all(evaluated[c] for c in children[v])]
        if not Vt:
            raise OracleError("cycle", "no activated vertex")
        S.append(Vt)               # already ascending global id (Z4)
        for v in Vt:
            evaluated[v] = True
        n_done += len(Vt)
    return S


def schedule(children):
    """(level[V], level_ptr[T+1], order[V]): V_t = {v : level(v)=t}, ascending id."""
    level = levels_recursive(children)
    T = int(level.max()) + 1 if len(level) else 0
    order = np.lexsort((np.arange(len(level)), level)).astype(np.int32)
    counts = np.bincount(level, minlength=T)
    level_ptr = np.zeros(T + 1, dtype=np.int32)
    level_ptr[1:] = np.cumsum(counts)
    return level, level_ptr, order


# ---------------------------------------------------------------------------
# parameters (packed layout of include/cavs.h)
# ---------------------------------------------------------------------------
def unpack(cell, N, h, d, theta):
    t = np.asarray(theta, dtype=np.float64)
    P = {}
    o = 0
    if cell == TREE_LSTM:
        W = t[o:o + 4 * h * d].reshape(4 * h, d); o += 4 * h * d
        P["W_i"], P["W_f"], P["W_o"], P["W_u"] = W[0:h], W[h:2 * h], W[2 * h:3 * h], W[3 * h:4 * h]
        U = t[o:o + 3 * h * h].reshape(3 * h, h); o += 3 * h * h
        P["U_i"], P["U_o"], P["U_u"] = U[0:h], U[h:2 * h], U[2 * h:3 * h]
        P["U_f"] = t[o:o + h * h].reshape(h, h); o += h * h
        b = t[o:o + 4 * h]; o += 4 * h
        P["b_i"], P["b_f"], P["b_o"], P["b_u"] = b[0:h], b[h:2 * h], b[2 * h:3 * h], b[3 * h:4 * h]
    elif cell == TREE_FC:
        Wc = t[o:o + 2 * h * h].reshape(h, 2 * h); o += 2 * h * h
        P["W_l"], P["W_r"] = Wc[:, 0:h], Wc[:, h:2 * h]
        P["W_x"] = t[o:o + h * d].reshape(h, d); o += h * d
        P["b"] = t[o:o + h]; o += h
    else:
        raise ValueError(cell)
    assert o == t.size, (o, t.size)
    return P


def pack(cell, N, h, d, P):
    if cell == TREE_LSTM:
        parts = [P["W_i"], P["W_f"], P["W_o"], P["W_u"], P["U_i"], P["U_o"], P["U_u"], P["U_f"],
                 P["b_i"], P["b_f"], P["b_o"], P["b_u"]]
    else:
        parts = [np.concatenate([P["W_l"], P["W_r"]], axis=1), P["W_x"], P["b"]]
    return np.concatenate([np.asarray(p, dtype=np.float64).ravel() for p in parts])


# ---------------------------------------------------------------------------
# forward / backward: plain per-vertex recursive evaluation
# ---------------------------------------------------------------------------
@dataclass
class Tape:
    log: list          # evaluation order of global vertex ids
    st: list           # per-vertex saved values (dict)
    children: list


def _mv(accum):
    """Matrix-vector product: fp64 (default), or `accum="fp32"`: operands rounded to fp32 and the
    sum accumulated in fp32 (numpy's order) -- a second valid fp32 evaluation.  With the bf16
    emulation the operands are bf16-exact, so every product is exact and only the running sum
    rounds (the tensor cores' arithmetic).  Diagnostic only: it measures how much F amplifies
    summation-order rounding (reading R-chaos)."""
    if accum == "fp64":
        return lambda A, v: A @ v
    if accum == "fp32":
        cache = {}                     # fp32 images of the (bf16-exact) weight matrices

        def mv32(A, v):
            key = (A.__array_interface__["data"][0], A.shape, A.strides)
            if key not in cache:
                cache[key] = np.asarray(A, np.float32)
            return (cache[key] @ np.asarray(v, np.float32)).astype(np.float64)
        return mv32
    raise ValueError(accum)


def forward(cell, N, h, d, theta, graph_ptr, child_ptr, child_idx, x_row, x, emulate_bf16=False,
            bf16_hsum="rounded", accum="fp64"):
    """Returns (h_out[V,h] fp64, tape).  Evaluates F at every vertex after all its
    children (Fig. 5); each vertex exactly once (memo).  `bf16_hsum` only
    matters with emulate_bf16 (see the module header); `accum` selects _mv."""
    mv = _mv(accum)
    if bf16_hsum not in ("rounded", "exact"):
        raise ValueError(bf16_hsum)
    ch = validate(graph_ptr, child_ptr, child_idx, N)
    V = len(ch)
    P = unpack(cell, N, h, d, theta)
    q = bf16r if emulate_bf16 else (lambda a: a)
    Pq = {k: (q(v) if not k.startswith("b") else v) for k, v in P.items()}
    X = np.asarray(x, dtype=np.float64)
    st = [None] * V
    log = []
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 4 * V + 1000))

    def pull(v):                      # pull(): external input or zeros (Z2)
        r = int(x_row[v])
        return q(X[r]) if r >= 0 else np.zeros(d)

    def ev(v):
        if st[v] is not None:
            return
        for c in ch[v]:
            ev(c)
        xv = pull(v)
        if cell == TREE_LSTM:
            # gather(k) for k < N; missing children are zero (Z1)
            hk = [st[c]["h"] for c in ch[v]] + [np.zeros(h)] * (N - len(ch[v]))
            ck = [st[c]["c"] for c in ch[v]] + [np.zeros(h)] * (N - len(ch[v]))
            hkq = [q(a) for a in hk]
            # h~ = sum_k h_k (Fig. 5); bf16 emulation: Z11 rounds it as a GEMM operand,
            # reading R-lin keeps the exact sum of the rounded slots
            hs = sum(hk)
            if emulate_bf16:
                hs = sum(hkq)
                if bf16_hsum == "rounded":
                    hs = q(hs)
            i = sigmoid(mv(Pq["W_i"], xv) + mv(Pq["U_i"], hs) + P["b_i"])
            f = [sigmoid(mv(Pq["W_f"], xv) + mv(Pq["U_f"], hkq[k]) + P["b_f"]) for k in range(N)]
            o = sigmoid(mv(Pq["W_o"], xv) + mv(Pq["U_o"], hs) + P["b_o"])
            u = np.tanh(mv(Pq["W_u"], xv) + mv(Pq["U_u"], hs) + P["b_u"])
            c = i * u + sum(f[k] * ck[k] for k in range(N))
            hv = o * np.tanh(c)
            st[v] = dict(h=hv, c=c, i=i, f=f, o=o, u=u, hs=hs, hkq=hkq, ck=ck, x=xv)
        else:
            hl = st[ch[v][0]]["h"] if len(ch[v]) > 0 else np.zeros(h)
            hr = st[ch[v][1]]["h"] if len(ch[v]) > 1 else np.zeros(h)
            hlq, hrq = q(hl), q(hr)
            z = mv(Pq["W_l"], hlq) + mv(Pq["W_r"], hrq) + mv(Pq["W_x"], xv) + P["b"]
            hv = np.tanh(z)
            st[v] = dict(h=hv, hkq=[hlq, hrq], x=xv)
        log.append(v)                  # scatter/push: h is published

    try:
        for v in range(V):
            ev(v)
    finally:
        sys.setrecursionlimit(old)
    h_out = np.stack([st[v]["h"] for v in range(V)]) if V else np.zeros((0, h))
    return h_out, Tape(log=log, st=st, children=ch)


def backward(cell, N, h, d, theta, tape, x_row, n_x, gamma, emulate_bf16=False, accum="fp64"):
    """dL/dparams (packed, fp64) and dL/dx [n_x, d] for L = sum_v <Gamma_v, h_v>.
    Reverse evaluation order (Alg. 1 BACKWARD); all gradients accumulate.
    `accum`: the dH / dx products' arithmetic, see _mv."""
    mv = _mv(accum)
    P = unpack(cell, N, h, d, theta)
    q = bf16r if emulate_bf16 else (lambda a: a)
    Pq = {k: (q(v) if not k.startswith("b") else v) for k, v in P.items()}
    G = {k: np.zeros_like(v) for k, v in P.items()}
    st, ch = tape.st, tape.children
    V = len(st)
    dh = np.array(gamma, dtype=np.float64).reshape(V, h).copy()   # push's adjoint: dL/dh_push
    dc = np.zeros((V, h))
    dx = np.zeros((n_x, d))
    for v in reversed(tape.log):
        s = st[v]
        r = int(x_row[v])
        if cell == TREE_LSTM:
            i, o, u, f, c = s["i"], s["o"], s["u"], s["f"], s["c"]
            tc = np.tanh(c)
            dz_o = dh[v] * tc * o * (1 - o)
            dcb = dc[v] + dh[v] * o * (1 - tc * tc)
            dz_i = dcb * u * i * (1 - i)
            dz_u = dcb * i * (1 - u * u)
            dz_f = [dcb * s["ck"][k] * f[k] * (1 - f[k]) for k in range(N)]
            dz_i, dz_o, dz_u = q(dz_i), q(dz_o), q(dz_u)
            dz_f = [q(a) for a in dz_f]
            dhs = mv(Pq["U_i"].T, dz_i) + mv(Pq["U_o"].T, dz_o) + mv(Pq["U_u"].T, dz_u)
            for k, cv in enumerate(ch[v]):           # scatter = adjoint of gather
                dh[cv] += dhs + mv(Pq["U_f"].T, dz_f[k])
                dc[cv] += dcb * f[k]
            hs = s["hs"]
            G["U_i"] += np.outer(dz_i, hs); G["U_o"] += np.outer(dz_o, hs); G["U_u"] += np.outer(dz_u, hs)
            for k in range(N):
                G["U_f"] += np.outer(dz_f[k], s["hkq"][k])
            G["b_i"] += dz_i; G["b_o"] += dz_o; G["b_u"] += dz_u
            G["b_f"] += sum(dz_f)
            if r >= 0:                               # pull's adjoint = push to the external
                xv = s["x"]
                G["W_i"] += np.outer(dz_i, xv); G["W_o"] += np.outer(dz_o, xv)
                G["W_u"] += np.outer(dz_u, xv)
                for k in range(N):
                    G["W_f"] += np.outer(dz_f[k], xv)
                dx[r] += (mv(Pq["W_i"].T, dz_i) + mv(Pq["W_o"].T, dz_o) + mv(Pq["W_u"].T, dz_u)
                          + mv(Pq["W_f"].T, sum(dz_f)))
        else:
            dz = q(dh[v] * (1 - s["h"] ** 2))
            hlq, hrq = s["hkq"]
            if len(ch[v]) > 0:
                dh[ch[v][0]] += mv(Pq["W_l"].T, dz)
            if len(ch[v]) > 1:
                dh[ch[v][1]] += mv(Pq["W_r"].T, dz)
            G["W_l"] += np.outer(dz, hlq)
            G["W_r"] += np.outer(dz, hrq)
            G["b"] += dz
            if r >= 0:
                G["W_x"] += np.outer(dz, s["x"])
                dx[r] += mv(Pq["W_x"].T, dz)
    return pack(cell, N, h, d, G), dx


def lm_head(h_out, W_out, b_out, targets):
    """Next-word softmax head outside (F, G) (reading Z9), plain definition in fp64:
    logits_v = W_out h_v + b_out; L = sum over vertices with a target of
    logsumexp(logits_v) - logits_v[target_v].  Returns (L, dL/dh [V,h], dL/dW_out, dL/db_out);
    dL/dh is the cotangent Gamma that push's adjoint hands to F's backward."""
    H = np.asarray(h_out, dtype=np.float64)
    W = np.asarray(W_out, dtype=np.float64)
    b = np.asarray(b_out, dtype=np.float64)
    t = np.asarray(targets)
    logits = H @ W.T + b
    mx = logits.max(axis=1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(axis=1))
    has = t >= 0
    L = float(np.sum(lse[has] - logits[has, t[has]]))
    dl = np.exp(logits - lse[:, None])
    dl[has, t[has]] -= 1.0
    dl[~has] = 0.0
    return L, dl @ W, dl.T @ H, dl.sum(axis=0)


def loss(h_out, gamma):
    """External linear loss L = sum_v <Gamma_v, h_v> (reading Z9)."""
    return float(np.sum(np.asarray(h_out) * np.asarray(gamma, dtype=np.float64)))


def run(batch, emulate_bf16=False, with_backward=True, bf16_hsum="rounded", accum="fp64"):
    """Convenience: forward (+ backward) on a workloads.Batch-like object."""
    h_out, tape = forward(batch.cell, batch.N, batch.h, batch.d, batch.params, batch.graph_ptr,
                          batch.child_ptr, batch.child_idx, batch.x_row, batch.x,
                          emulate_bf16=emulate_bf16, bf16_hsum=bf16_hsum, accum=accum)
    if not with_backward:
        return h_out, None, None, tape
    dparams, dx = backward(batch.cell, batch.N, batch.h, batch.d, batch.params, tape, batch.x_row,
                           batch.x.shape[0], batch.gamma, emulate_bf16=emulate_bf16, accum=accum)
    return h_out, dparams, dx, tape
