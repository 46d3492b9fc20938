"""CPU oracle of the COMM-RAND mini-batch hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2504_18082_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain single-threaded C, one
function per step, each citing the paper passage it follows); this module only
marshals numpy arrays through ctypes and composes the per-hop calls in the
order of Alg. 1.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): Philox KAT, mulhi64 closed
forms, brute-force graph prep, Knob-1 invariants + chi^2, the exact
without-replacement law of Knob-2 by enumeration + chi^2, brute-force relabel,
fp64 closed forms for the aggregate.  See DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]

MODE_RAND, MODE_NORAND, MODE_COMM, MODE_COMM_STATIC = 0, 1, 2, 3

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO + ".tmp", _SRC])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, I64, I32, U32, U64, D = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_double)
        L.or_philox4x32_10.argtypes = [P, P, P]
        L.or_mulhi64.argtypes = [U64, U64]
        L.or_mulhi64.restype = U64
        L.or_graph_prep.argtypes = [I64, P, P, P, I32, P, P, P]
        L.or_graph_prep.restype = ctypes.c_int
        L.or_community_order.argtypes = [I64, P, P, P, P, P, P, P, P]
        L.or_community_order.restype = ctypes.c_int
        L.or_order_roots.argtypes = [I64, P, P, I32, I32, D, U64, U32, P]
        L.or_order_roots.restype = ctypes.c_int
        L.or_sample_hop.argtypes = [P, I64, P, P, P, P, I32, D, U64, I32, U32, P, P, I64, I32]
        L.or_sample_hop.restype = I64
        L.or_relabel_hop.argtypes = [P, I64, I64, P, I64, P, P]
        L.or_relabel_hop.restype = I64
        L.or_gather.argtypes = [P, I64, P, I64, I32, P, I64]
        L.or_sage_mean.argtypes = [P, P, I64, P, I64, P, I32, P, I64, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------- O1
def philox(ctr, key) -> np.ndarray:
    c, k = _c(ctr, np.uint32), _c(key, np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def mulhi64(r: int, n: int) -> int:
    return int(lib().or_mulhi64(r, n))


# ---------------------------------------------------------------- a0
class Prep:
    def __init__(self, indptr, indices, comm, num_comm):
        self.indptr = _c(indptr, np.int64)
        self.indices = _c(indices, np.int32)
        self.comm = _c(comm, np.int32)
        self.num_comm = int(num_comm)
        n = self.indptr.shape[0] - 1
        self.cbeg = np.zeros(self.num_comm + 1, dtype=np.int32)
        self.lo = np.zeros(n, dtype=np.uint32)
        self.hi = np.zeros(n, dtype=np.uint32)
        self.status = lib().or_graph_prep(n, _p(self.indptr), _p(self.indices), _p(self.comm),
                                          self.num_comm, _p(self.cbeg), _p(self.lo), _p(self.hi))

    @property
    def num_nodes(self):
        return self.indptr.shape[0] - 1


def graph_prep(bundle) -> Prep:
    return Prep(bundle.indptr, bundle.indices, bundle.comm, bundle.cfg.num_communities)


# ---------------------------------------------------------------- a1
def order_roots(train, comm, num_comm, mode, mix=0.0, seed=42, epoch=0) -> np.ndarray:
    t, cm = _c(train, np.int32), _c(comm, np.int32)
    out = np.zeros(t.shape[0], dtype=np.int32)
    rc = lib().or_order_roots(t.shape[0], _p(t), _p(cm), int(num_comm), int(mode), float(mix),
                              int(seed), int(epoch), _p(out))
    if rc != 0:
        raise ValueError("or_order_roots failed (empty train set?)")
    return out


def community_order(indptr, indices, comm):
    """NEXT-2 (iii): (perm new->old, inv old->new, indptr, indices, comm) of the community-
    ordered relabelling of an arbitrary graph (reading R25)."""
    ip, ix, cm = _c(indptr, np.int64), _c(indices, np.int32), _c(comm, np.int32)
    n = ip.shape[0] - 1
    perm, inv = np.zeros(n, np.int32), np.zeros(n, np.int32)
    ip2, ix2, cm2 = np.zeros(n + 1, np.int64), np.zeros(max(1, ix.shape[0]), np.int32), np.zeros(n, np.int32)
    lib().or_community_order(n, _p(ip), _p(ix), _p(cm), _p(perm), _p(inv), _p(ip2), _p(ix2), _p(cm2))
    return perm, inv, ip2, ix2[: ix.shape[0]], cm2


def batch_roots(order: np.ndarray, batch_size: int, b: int) -> np.ndarray:
    """Alg. 1 line 2 "Divide nodes across mini-batches": consecutive B-slices, last partial kept."""
    return order[b * batch_size: min((b + 1) * batch_size, order.shape[0])]


# ---------------------------------------------------------------- a2
LAW_A, LAW_SLOT = 0, 1   # Knob-2 laws: successive weighted w/o replacement (R1) / slot (R23)


def sample_hop(prep: Prep, dst_nodes, fanout, p, seed, hop, batch, law=LAW_A):
    d = _c(dst_nodes, np.int32)
    cap = d.shape[0] * int(fanout)
    indptr_h = np.zeros(d.shape[0] + 1, dtype=np.int64)
    nbr = np.zeros(max(1, cap), dtype=np.int32)
    e = lib().or_sample_hop(_p(d), d.shape[0], _p(prep.indptr), _p(prep.indices), _p(prep.lo),
                            _p(prep.hi), int(fanout), float(p), int(seed), int(hop), int(batch),
                            _p(indptr_h), _p(nbr), cap, int(law))
    assert e >= 0
    return indptr_h, nbr[:e]


# ---------------------------------------------------------------- a3
def relabel_hop(nodes_prefix, nbr, num_nodes, scratch=None):
    n_dst = nodes_prefix.shape[0]
    cap = n_dst + nbr.shape[0]
    nodes = np.zeros(max(1, cap), dtype=np.int32)
    nodes[:n_dst] = nodes_prefix
    local = np.zeros(max(1, nbr.shape[0]), dtype=np.int32)
    m = scratch if scratch is not None else np.full(num_nodes, -1, dtype=np.int32)
    nb = _c(nbr, np.int32)
    n_next = lib().or_relabel_hop(_p(nodes), n_dst, cap, _p(nb), nb.shape[0], _p(local), _p(m))
    assert n_next >= 0
    return nodes[:n_next], local[: nb.shape[0]]


def sample_blocks(prep: Prep, roots, fanouts, p, seed, batch, scratch=None, law=LAW_A):
    """Alg. 1 lines 4-5 for one batch: hop h = 0..L-1 expands nodes[0:n_h).

    Returns dict: nodes (nested prefixes), n (list n_0..n_L), e (list e_0..e_{L-1}),
    indptr[h] (int64 [n_h+1]), indices[h] (local ids), nbr[h] (global ids)."""
    nodes = _c(roots, np.int32)
    n, e, indptr, indices, nbrs = [nodes.shape[0]], [], [], [], []
    if scratch is None:
        scratch = np.full(prep.num_nodes, -1, dtype=np.int32)
    for h, f in enumerate(fanouts):
        ip, nbr = sample_hop(prep, nodes, f, p, seed, h, batch, law)
        nodes, local = relabel_hop(nodes, nbr, prep.num_nodes, scratch)
        indptr.append(ip)
        indices.append(local)
        nbrs.append(nbr)
        e.append(nbr.shape[0])
        n.append(nodes.shape[0])
    return {"nodes": nodes, "n": n, "e": e, "indptr": indptr, "indices": indices, "nbr": nbrs}


# ---------------------------------------------------------------- a4
def gather(nodes, X, F=None) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float32)
    F = X.shape[1] if F is None else F
    nd = _c(nodes, np.int32)
    out = np.zeros((nd.shape[0], F), dtype=np.float32)
    lib().or_gather(_p(nd), nd.shape[0], _p(X), X.shape[1], int(F), _p(out), F)
    return out


# ---------------------------------------------------------------- a5
def sage_mean(indptr_h, idx, Xsrc, F=None, src_map=None):
    Xsrc = np.ascontiguousarray(Xsrc, dtype=np.float32)
    F = Xsrc.shape[1] if F is None else F
    ip, ix = _c(indptr_h, np.int64), _c(idx, np.int32)
    n_dst = ip.shape[0] - 1
    out = np.zeros((n_dst, F), dtype=np.float32)
    out64 = np.zeros((n_dst, F), dtype=np.float64)
    sm = None if src_map is None else _c(src_map, np.int32)
    lib().or_sage_mean(_p(ip), _p(ix), n_dst, _p(Xsrc), Xsrc.shape[1], _p(sm), int(F), _p(out), F,
                       _p(out64))
    return out, out64


def run_batch(prep: Prep, X, F, roots, fanouts, p, seed, batch, scratch=None, law=LAW_A):
    """One whole hot-path step (a2-a5) for one batch, as the oracle defines it."""
    blk = sample_blocks(prep, roots, fanouts, p, seed, batch, scratch, law)
    L = len(fanouts)
    Xin = gather(blk["nodes"], X, F)
    H, H64 = sage_mean(blk["indptr"][L - 1], blk["indices"][L - 1], Xin, F)
    blk.update({"X_in": Xin, "H": H, "H64": H64})
    return blk


# ---------------------------------------------------------------- NEXT-4: first SAGEConv layer
def sage_conv(X_dst, H, W_self, W_neigh, bias=None, relu=False) -> np.ndarray:
    """Forward of the input-side GraphSAGE layer (reading R26), fp64.

    Eq. (1) (the layer update X^{l+1} = sigma(A' X^l W^l)) in the
    GraphSAGE-mean form its footnote points to (Hamilton et al.; the paper trains
    GraphSAGE, hidden dim 256):

        Y[d, :] = sigma( X_dst[d, :] @ W_self + H[d, :] @ W_neigh + bias )

    X_dst = X_in[0:n_dst] (the dst nodes are the prefix of the src nodes, reading R8),
    H = the a5 mean aggregate of the same rows, W_self / W_neigh are F x Fo (row-major,
    Y = X W as in Eq. (1)), sigma = ReLU when relu else identity.  Exact fp64 on the given
    values: the bf16 operand rounding of the GPU kernel is NOT modelled here; the parity
    tests bound it (R26).  Test infrastructure only (see the module header).
    """
    X = np.asarray(X_dst, dtype=np.float64)
    Hn = np.asarray(H, dtype=np.float64)
    Ws = np.asarray(W_self, dtype=np.float64)
    Wn = np.asarray(W_neigh, dtype=np.float64)
    Y = X @ Ws + Hn @ Wn
    if bias is not None:
        Y = Y + np.asarray(bias, dtype=np.float64)[None, :]
    if relu:
        Y = np.maximum(Y, 0.0)
    return Y


def sage_conv_backward(X_dst, H, dY, Y=None, relu=False):
    """Weight gradients of the input-side GraphSAGE layer (NEXT-4 backward, reading R27), fp64.

    For Y = sigma(Z), Z = X_dst W_self + H W_neigh + b (sage_conv) and an upstream gradient dY:
    dZ = dY * sigma'(Z) (ReLU: 1[Y > 0], the decision taken on the given Y; identity: 1),
    dW_self = X_dst^T dZ, dW_neigh = H^T dZ, db = sum_d dZ[d, :] -- the chain rule on Eq. (1)
    (training learns W^l by minimising the loss).  X_dst and H of the first
    layer are inputs (features), so no gradient flows to them.  Returns (dW_self, dW_neigh, db).
    """
    X = np.asarray(X_dst, dtype=np.float64)
    Hn = np.asarray(H, dtype=np.float64)
    dZ = np.asarray(dY, dtype=np.float64)
    if relu:
        dZ = dZ * (np.asarray(Y, dtype=np.float64) > 0)
    return X.T @ dZ, Hn.T @ dZ, dZ.sum(axis=0)


def gcn_conv(indptr_h, idx, X_in, W, bias=None, relu=False) -> np.ndarray:
    """GCN form of the input-side layer (NEXT-4 variant, reading R28), fp64.

    Eq. (1) X^{l+1} = sigma(A' X^l W) with A' "the normalized and regularized
    adjacency matrix", taken on the sampled block of hop L-1 as the row-normalised adjacency with
    a self loop, A' = (D + I)^{-1} (A + I): row d of A' X_in is (X_in[d] + sum_{e in row d}
    X_in[idx[e]]) / (deg_d + 1) -- dst node d is src node d (the dst list is the prefix of the
    src list, reading R8).  Y = sigma(A' X_in W + bias), W F x Fo row-major.
    """
    ip = np.asarray(indptr_h, dtype=np.int64)
    ix = np.asarray(idx, dtype=np.int64)
    X = np.asarray(X_in, dtype=np.float64)
    n_dst = ip.shape[0] - 1
    deg = np.diff(ip)
    S = X[:n_dst].copy()
    np.add.at(S, np.repeat(np.arange(n_dst), deg), X[ix])
    Y = (S / (deg + 1.0)[:, None]) @ np.asarray(W, dtype=np.float64)
    if bias is not None:
        Y = Y + np.asarray(bias, dtype=np.float64)[None, :]
    if relu:
        Y = np.maximum(Y, 0.0)
    return Y


def gcn_aggregate64(indptr_h, idx, X_in) -> np.ndarray:
    """Row d of A' X_in for the GCN form (reading R28): (X_in[d] + sum_{e in row d}
    X_in[idx[e]]) / (deg_d + 1), fp64 -- the aggregate gcn_conv multiplies by W."""
    ip = np.asarray(indptr_h, dtype=np.int64)
    ix = np.asarray(idx, dtype=np.int64)
    X = np.asarray(X_in, dtype=np.float64)
    n_dst = ip.shape[0] - 1
    deg = np.diff(ip)
    S = X[:n_dst].copy()
    np.add.at(S, np.repeat(np.arange(n_dst), deg), X[ix])
    return S / (deg + 1.0)[:, None]


def gcn_conv_backward(indptr_h, idx, X_in, dY, Y=None, relu=False):
    """Weight gradients of the GCN form of the layer (NEXT-4, reading R35), fp64.

    For Y = sigma(Z), Z = G W + b with G = A' X_in (gcn_conv, reading R28) and an upstream dY:
    dZ = dY * sigma'(Z) (ReLU: 1[Y > 0] on the given Y), dW = G^T dZ, db = sum_d dZ[d, :] -- the
    chain rule on Eq. (1); the features get no gradient.  Returns (dW, db).
    """
    G = gcn_aggregate64(indptr_h, idx, X_in)
    dZ = np.asarray(dY, dtype=np.float64)
    if relu:
        dZ = dZ * (np.asarray(Y, dtype=np.float64) > 0)
    return G.T @ dZ, dZ.sum(axis=0)


def sage_mean64(indptr_h, idx, Xsrc) -> np.ndarray:
    """a5's mean (reading R12: neighbours only, 0 for an empty row) on fp64 inputs, for
    the hidden layers of the model (reading R29), whose inputs are the previous layer's outputs:
    H[d] = (sum_{e in row d} Xsrc[idx[e]]) / deg_d."""
    ip = np.asarray(indptr_h, dtype=np.int64)
    X = np.asarray(Xsrc, dtype=np.float64)
    n = ip.shape[0] - 1
    deg = np.diff(ip)
    H = np.zeros((n, X.shape[1]), dtype=np.float64)
    np.add.at(H, np.repeat(np.arange(n), deg), X[np.asarray(idx, dtype=np.int64)])
    nz = deg > 0
    H[nz] /= deg[nz, None]
    return H


def sage_mean_backward(indptr_h, idx, dH, n_src) -> np.ndarray:
    """Backward of a5's mean through the transposed block (NEXT-4 "transposed-block scatter-add",
    reading R30), fp64: H = M X with M[d, idx[e]] += 1/deg_d for e in row d (R12), so
    dX = M^T dH, i.e. dX[idx[e], :] += dH[d, :] / deg_d for every edge e of row d; rows of X that
    no edge references get 0.  Returns dX [n_src, F]."""
    ip = np.asarray(indptr_h, dtype=np.int64)
    G = np.asarray(dH, dtype=np.float64)
    deg = np.diff(ip)
    dX = np.zeros((int(n_src), G.shape[1]), dtype=np.float64)
    rows = np.repeat(np.arange(ip.shape[0] - 1), deg)
    np.add.at(dX, np.asarray(idx, dtype=np.int64), G[rows] / deg[rows, None])
    return dX


def sage_hidden_input_grad(indptr_h, idx, dZ, W_self, W_neigh, n_src) -> np.ndarray:
    """Gradient into a hidden layer's input Yp (NEXT-4 backward of layers 2-3, reading R32), fp64:
    the layer (R29) reads Yp through its dst-prefix rows (Yp[d] W_self, d < n_dst: the dst list
    is the prefix of the src list, R8) and through the neighbour mean (M Yp) W_neigh, so by the
    chain rule dYp = P^T (dZ W_self^T) + M^T (dZ W_neigh^T), with M^T = sage_mean_backward (R30).
    dZ = dY * sigma'(Z) is an input.  Returns dYp [n_src, Fin]."""
    G = np.asarray(dZ, dtype=np.float64)
    Ws = np.asarray(W_self, dtype=np.float64)
    Wn = np.asarray(W_neigh, dtype=np.float64)
    dX = sage_mean_backward(indptr_h, idx, G @ Wn.T, n_src)
    dX[:G.shape[0]] += G @ Ws.T
    return dX


def softmax_xent(Y, labels):
    """The training loss (NEXT-4, reading R33), fp64: PAPER.md P:503 trains the layer parameters
    "by minimizing the loss between the labels of all labeled nodes and the node embeddings of
    the last layer"; the loss of DGL's GraphSAGE node classification is the softmax cross-entropy,
    averaged over the batch's n roots:
        loss = (1/n) sum_i [ log sum_c exp(Y[i, c]) - Y[i, label_i] ],
        dY[i, c] = (exp(Y[i, c]) / sum_c' exp(Y[i, c']) - 1[c == label_i]) / n.
    Y: [n, C] logits; labels: [n] ints in [0, C).  Returns (loss, dY)."""
    Y = np.asarray(Y, dtype=np.float64)
    lab = np.asarray(labels, dtype=np.int64)
    n = Y.shape[0]
    if n == 0:
        return 0.0, np.zeros_like(Y)
    m = Y.max(axis=1, keepdims=True)
    e = np.exp(Y - m)
    s = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(s))[:, 0]
    loss = float(np.mean(lse - Y[np.arange(n), lab]))
    dY = e / s
    dY[np.arange(n), lab] -= 1.0
    return loss, dY / n


def adam_step(w, g, m, v, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=5e-4):
    """One optimizer step (NEXT-4, reading R34), fp64: Adam with L2 weight decay added to the
    gradient (torch.optim.Adam semantics; DGL's GraphSAGE defaults lr = 1e-3, weight decay 5e-4,
    PAPER.md P:774):  g' = g + wd w;  m = b1 m + (1 - b1) g';  v = b2 v + (1 - b2) g'^2;
    w = w - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps).  Returns new (w, m, v)."""
    w = np.asarray(w, dtype=np.float64)
    gp = np.asarray(g, dtype=np.float64) + weight_decay * w
    m = beta1 * np.asarray(m, dtype=np.float64) + (1.0 - beta1) * gp
    v = beta2 * np.asarray(v, dtype=np.float64) + (1.0 - beta2) * gp * gp
    mh = m / (1.0 - beta1 ** step)
    vh = v / (1.0 - beta2 ** step)
    return w - lr * mh / (np.sqrt(vh) + eps), m, v
