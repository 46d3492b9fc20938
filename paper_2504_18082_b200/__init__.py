"""B200-native COMM-RAND mini-batch hot path (arXiv 2504.18082) -- Python binding.

Thin ctypes layer over ``libcmb.so`` (the C ABI declared in ``include/cmb.h``).
It only marshals arguments: PyTorch supplies device memory (every buffer and
workspace is a torch tensor) and the current CUDA stream; every step of the
path runs in the library's sm_100a kernels.  There is no CPU fallback: if the
extension is missing or the device is not a B200 the calls raise.

Public API (names follow the C ABI):
  Graph(...)                       a0  cmb_load_graph
  order_roots(graph, train, ...)   a1  cmb_order_roots
  Sampler(graph, ...).sample(...)  a2+a3 cmb_sample_blocks
  gather_features(...)             a4  cmb_gather_features
  sage_mean_aggregate(...)         a5  cmb_sage_mean_aggregate
  Sampler.gather_aggregate(...)    a4+a5 cmb_gather_aggregate
  MiniBatchPipeline                the whole step (Alg. 1)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CMB_LIB_PATH") or os.path.join(_HERE, "libcmb.so")  # override: A/B builds
MAX_HOPS = 8
MAX_FANOUT = 32

ROOTS_RAND, ROOTS_NORAND, ROOTS_COMM, ROOTS_COMM_STATIC = 0, 1, 2, 3
_MODES = {"rand": ROOTS_RAND, "norand": ROOTS_NORAND, "comm": ROOTS_COMM,
          "comm_static": ROOTS_COMM_STATIC}

STATUS = {0: "CMB_OK", 1: "CMB_ERR_INVALID_ARGUMENT", 2: "CMB_ERR_INVALID_GRAPH",
          3: "CMB_ERR_NOT_COMMUNITY_ORDERED", 4: "CMB_ERR_CAPACITY", 5: "CMB_ERR_CUDA",
          6: "CMB_ERR_UNSUPPORTED_DEVICE", 7: "CMB_ERR_INVALID_INPUT"}

# C ABI symbols (include/cmb.h); tests check the library exports all of them.
SYMBOLS = ["cmb_graph_workspace_bytes", "cmb_load_graph", "cmb_free_graph", "cmb_graph_arrays",
           "cmb_order_roots_workspace_bytes", "cmb_order_roots", "cmb_blocks_capacity",
           "cmb_sample_workspace_bytes", "cmb_sample_blocks", "cmb_sample_blocks_law",
           "cmb_sample_blocks_multi",
           "cmb_gather_features",
           "cmb_sage_mean_aggregate", "cmb_gather_aggregate", "cmb_gather_aggregate_multi",
           "cmb_shard_plan_workspace_bytes",
           "cmb_shard_plan", "cmb_gather_rows", "cmb_scatter_rows",
           "cmb_gather_aggregate_sharded", "cmb_ipc_export", "cmb_ipc_open", "cmb_ipc_close",
           "cmb_step_group", "cmb_feature_cache_bytes", "cmb_feature_cache_init",
           "cmb_community_order_workspace_bytes", "cmb_community_order",
           "cmb_cache_gather_aggregate",
           "cmb_sage_weights_bytes", "cmb_sage_pack_weights", "cmb_sage_layer_forward",
           "cmb_sage_backward_workspace_bytes", "cmb_sage_layer_backward",
           "cmb_gcn_weights_bytes", "cmb_gcn_pack_weights", "cmb_gcn_layer_forward",
           "cmb_gcn_layer_backward",
           "cmb_sage_hidden_weights_bytes", "cmb_sage_hidden_pack_weights",
           "cmb_sage_hidden_forward", "cmb_sage_mean_backward",
           "cmb_sage_hidden_backward_workspace_bytes", "cmb_sage_hidden_backward",
           "cmb_sage_hidden_weights_t_bytes", "cmb_sage_hidden_pack_weights_t",
           "cmb_sage_hidden_input_grad", "cmb_softmax_xent", "cmb_adam_step",
           "cmb_sage_saved_a_bytes", "cmb_sage_layer_forward_save", "cmb_sage_layer_backward_saved",
           "cmb_adam_step_pack", "cmb_adam_step_pack_dev", "cmb_sage_dense_weights_bytes", "cmb_sage_dense_workspace_bytes",
           "cmb_sage_dense_pack_weights", "cmb_sage_dense_forward", "cmb_sage_dense_backward",
           "cmb_get_device_status",
           "cmb_status_string", "cmb_last_error_message", "cmb_version"]


class CmbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class GraphDesc(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("num_edges", ctypes.c_int64),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p),
                ("community", ctypes.c_void_p), ("num_communities", ctypes.c_int32),
                ("features", ctypes.c_void_p), ("feat_dim", ctypes.c_int32),
                ("feat_ld", ctypes.c_int64), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("validate", ctypes.c_int32)]


class Blocks(ctypes.Structure):
    _fields_ = [("nodes", ctypes.c_void_p), ("nodes_cap", ctypes.c_int64),
                ("indptr", ctypes.c_void_p * MAX_HOPS), ("indices", ctypes.c_void_p * MAX_HOPS),
                ("indices_cap", ctypes.c_int64 * MAX_HOPS), ("new_src_mask", ctypes.c_void_p),
                ("last_src_ids", ctypes.c_void_p), ("sizes", ctypes.c_void_p),
                ("dst_order", ctypes.c_void_p)]


class Batch(ctypes.Structure):
    _fields_ = [("roots", ctypes.c_void_p), ("n_roots", ctypes.c_int64),
                ("batch_id", ctypes.c_uint32), ("out", ctypes.POINTER(Blocks)),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


class LayerPack(ctypes.Structure):
    """cmb_layer_pack (include/cmb.h)."""
    _fields_ = [("offset", ctypes.c_int64), ("in_dim", ctypes.c_int32), ("out_dim", ctypes.c_int32),
                ("img", ctypes.c_void_p), ("img_t", ctypes.c_void_p), ("dense", ctypes.c_int32)]


class FeatureCacheDesc(ctypes.Structure):
    _fields_ = [("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("num_nodes", ctypes.c_int64), ("capacity", ctypes.c_int64),
                ("max_rows", ctypes.c_int64), ("max_edges", ctypes.c_int64),
                ("host_x", ctypes.c_void_p), ("host_ld", ctypes.c_int64),
                ("cache_rows", ctypes.c_void_p), ("cache_ld", ctypes.c_int64)]


class BatchFeatures(ctypes.Structure):
    _fields_ = [("x_in", ctypes.c_void_p), ("x_in_ld", ctypes.c_int64), ("h_out", ctypes.c_void_p),
                ("h_ld", ctypes.c_int64), ("n_last_dst_cap", ctypes.c_int64),
                ("nodes_cap", ctypes.c_int64)]


MAX_BATCHES_PER_LAUNCH = 8
# batches per sampler launch of the benchmarked step (bench.py default; products: 166 us per batch
# at 6 vs 169 at 4 and 171 at 8 -- 148 SMs split into 6 virtual grids of 24 blocks)
DEFAULT_BATCHES_PER_LAUNCH = 6
LAW_A, LAW_SLOT = 0, 1  # Knob-2 laws (include/cmb.h cmb_sample_law)


def sage_mean_backward(indptr: torch.Tensor, indices: torch.Tensor, n_dst: torch.Tensor,
                       dh: torch.Tensor, dx: torch.Tensor, feat_dim: Optional[int] = None):
    """NEXT-4 (R30): dx[indices[e]] += dh[d] / deg_d over the transposed block (adds into dx).
    n_dst: device int64 [1] count (e.g. a Sampler's sizes[h:h+1])."""
    F = int(dh.shape[1] if feat_dim is None else feat_dim)
    _check(lib().cmb_sage_mean_backward(_ptr(indptr), _ptr(indices), _ptr(n_dst),
                                        int(indptr.shape[0] - 1), _ptr(dh), dh.stride(0), F,
                                        _ptr(dx), dx.stride(0), _stream()))
    return dx


def _law(law) -> int:
    if isinstance(law, str):
        return {"a": LAW_A, "slot": LAW_SLOT}[law.lower()]
    return int(law)
_lib = None


def lib():
    """Load libcmb.so; raise loudly if it was not built (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32, U32, U64, D, SZ = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double,
                                        ctypes.c_size_t)
        sig = {
            "cmb_graph_workspace_bytes": (SZ, [I64, I32]),
            "cmb_load_graph": (I32, [ctypes.POINTER(GraphDesc), P, ctypes.POINTER(P)]),
            "cmb_free_graph": (I32, [P]),
            "cmb_graph_arrays": (I32, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
            "cmb_order_roots_workspace_bytes": (SZ, [I64, I32]),
            "cmb_order_roots": (I32, [P, P, I64, I32, D, U64, U32, P, P, SZ, P]),
            "cmb_blocks_capacity": (None, [I64, P, I32, I64, P, P]),
            "cmb_sample_workspace_bytes": (SZ, [I64, P, I32, I64]),
            "cmb_sample_blocks": (I32, [P, P, I64, P, I32, D, U64, U32, ctypes.POINTER(Blocks), P,
                                        SZ, P]),
            "cmb_sample_blocks_law": (I32, [P, P, I64, P, I32, D, I32, U64, U32,
                                            ctypes.POINTER(Blocks), P, SZ, P]),
            "cmb_sample_blocks_multi": (I32, [P, ctypes.POINTER(Batch), I32, P, I32, D, I32, U64,
                                              P]),
            "cmb_gather_features": (I32, [P, P, P, I64, P, I64, P]),
            "cmb_sage_mean_aggregate": (I32, [P, P, P, I64, P, I64, P, I32, P, I64, P]),
            "cmb_gather_aggregate": (I32, [P, ctypes.POINTER(Blocks), I32, I64, I64, P, I64, P,
                                           I64, P]),
            "cmb_shard_plan_workspace_bytes": (SZ, [I64]),
            "cmb_shard_plan": (I32, [P, P, I64, I64, I32, P, P, P, P, SZ, P]),
            "cmb_gather_rows": (I32, [P, I64, I64, I32, P, P, I64, P, I64, P]),
            "cmb_scatter_rows": (I32, [P, I64, P, P, I64, I32, P, I64, P]),
            "cmb_gather_aggregate_sharded": (I32, [P, ctypes.POINTER(Blocks), I32, I64, I64, P,
                                                   I32, I64, I64, I32, P, I64, P, I64, P]),
            "cmb_ipc_export": (I32, [P, P, ctypes.POINTER(ctypes.c_uint64)]),
            "cmb_ipc_open": (I32, [P, ctypes.c_uint64, ctypes.POINTER(P), ctypes.POINTER(P)]),
            "cmb_ipc_close": (I32, [P]),
            "cmb_step_group": (I32, [P, ctypes.POINTER(Batch), ctypes.POINTER(BatchFeatures), I32,
                                     P, I32, D, I32, U64, P, P]),
            "cmb_feature_cache_bytes": (SZ, [I64, I64, I64, I64]),
            "cmb_community_order_workspace_bytes": (SZ, [I64, I64]),
            "cmb_community_order": (I32, [P, P, P, I64, I64, I32, P, P, P, P, P, P, SZ, P]),
            "cmb_feature_cache_init": (I32, [P, SZ, I64, I64, I64, I64, P]),
            "cmb_cache_gather_aggregate": (I32, [P, ctypes.POINTER(Blocks), I32, I64, I64,
                                                 ctypes.POINTER(FeatureCacheDesc), I32,
                                                 ctypes.c_uint32, P, I64, P, I64, P, P]),
            "cmb_sage_weights_bytes": (SZ, [I32, I32]),
            "cmb_sage_pack_weights": (I32, [P, P, I32, I32, P, SZ, P]),
            "cmb_sage_layer_forward": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, P, I32, I32,
                                             I32, P, I64, P]),
            "cmb_sage_backward_workspace_bytes": (SZ, [I32, I32]),
            "cmb_gcn_weights_bytes": (SZ, [I32, I32]),
            "cmb_sage_hidden_weights_bytes": (SZ, [I32, I32]),
            "cmb_sage_mean_backward": (I32, [P, P, P, I64, P, I64, I32, P, I64, P]),
            "cmb_sage_hidden_pack_weights": (I32, [P, P, I32, I32, P, SZ, P]),
            "cmb_sage_hidden_forward": (I32, [ctypes.POINTER(Blocks), I32, I64, P, I64, I32, P, P,
                                              I32, I32, I32, P, I64, P]),
            "cmb_gcn_pack_weights": (I32, [P, I32, I32, P, SZ, P]),
            "cmb_gcn_layer_forward": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, P, I32, I32,
                                            I32, P, I64, P]),
            "cmb_sage_layer_backward": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, I64, I32, P,
                                              I64, I32, P, P, P, SZ, P]),
            "cmb_gcn_layer_backward": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, I64, I32, P,
                                             I64, I32, P, P, P, SZ, P]),
            "cmb_sage_hidden_backward_workspace_bytes": (SZ, [I32, I32]),
            "cmb_sage_hidden_backward": (I32, [ctypes.POINTER(Blocks), I32, I64, P, I64, I32, P,
                                               I64, I32, P, I64, I32, P, P, P, SZ, P, I64, P]),
            "cmb_sage_hidden_weights_t_bytes": (SZ, [I32, I32]),
            "cmb_sage_saved_a_bytes": (SZ, [I32, I64]),
            "cmb_adam_step_pack": (I32, [P, P, P, P, I64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, I32,
                                         ctypes.POINTER(LayerPack), I32, P]),
            "cmb_adam_step_pack_dev": (I32, [P, P, P, P, I64, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             P, ctypes.POINTER(LayerPack), I32, P]),
            "cmb_sage_layer_forward_save": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, P, I32,
                                                  I32, I32, P, I64, P, SZ, P]),
            "cmb_sage_layer_backward_saved": (I32, [P, ctypes.POINTER(Blocks), I32, I64, P, SZ, P,
                                                    I64, I32, P, I64, I32, P, P, P, SZ, P]),
            "cmb_softmax_xent": (I32, [P, I64, P, P, P, I64, I32, P, I64, I32, P, P, P, P]),
            "cmb_adam_step": (I32, [P, P, P, P, I64, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double, I32, P]),
            "cmb_sage_hidden_pack_weights_t": (I32, [P, P, I32, I32, P, SZ, P]),
            "cmb_sage_hidden_input_grad": (I32, [ctypes.POINTER(Blocks), I32, I64, I64, P, I64, I32,
                                                 P, I32, P, I64, P, I64, P]),
            "cmb_sage_dense_weights_bytes": (SZ, [I32, I32]),
            "cmb_sage_dense_workspace_bytes": (SZ, [I64, I32, I32]),
            "cmb_sage_dense_pack_weights": (I32, [P, P, I32, I32, P, SZ, P]),
            "cmb_sage_dense_forward": (I32, [P, I64, P, I64, P, I64, I32, P, P, I32, I32, I32, P,
                                             I64, P, SZ, P]),
            "cmb_sage_dense_backward": (I32, [P, I64, P, I64, P, I64, I32, P, I64, I32, P, I64,
                                              I32, P, P, P, SZ, P]),
            "cmb_get_device_status": (I32, [P, P]),
            "cmb_status_string": (ctypes.c_char_p, [I32]),
            "cmb_last_error_message": (ctypes.c_char_p, []),
            "cmb_version": (ctypes.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise CmbError(code, lib().cmb_last_error_message().decode())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev_tensor(t, dtype, device):
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    return t.to(device=device, dtype=dtype).contiguous()


def _grad_out(dw, db, F, fo, device):
    """Gradient outputs of a layer backward: caller-given views ([2, F, fo] and [fo] fp32,
    contiguous) or fresh tensors."""
    if dw is None:
        dw = torch.empty(2, F, fo, dtype=torch.float32, device=device)
    if db is None:
        db = torch.empty(fo, dtype=torch.float32, device=device)
    if tuple(dw.shape) != (2, F, fo) or not dw.is_contiguous() or dw.dtype != torch.float32 or \
            tuple(db.shape) != (fo,) or db.dtype != torch.float32:
        raise ValueError("dw must be contiguous fp32 [2, F, out_dim], db fp32 [out_dim]")
    return dw, db


def softmax_xent(logits: torch.Tensor, node_labels: torch.Tensor, nodes: torch.Tensor,
                 n_dev: torch.Tensor, num_classes: int, dy: torch.Tensor, loss: torch.Tensor,
                 status: Optional[torch.Tensor] = None, row_loss: Optional[torch.Tensor] = None):
    """NEXT-4 loss (R33): softmax cross-entropy over the batch's roots (the prefix of `nodes`,
    n = n_dev[0]) -> loss (device fp64 [1]) and dY (bf16, columns >= num_classes zero)."""
    if row_loss is None or row_loss.numel() < dy.shape[0]:
        row_loss = torch.empty(max(1, dy.shape[0]), dtype=torch.float64, device=dy.device)
    _check(lib().cmb_softmax_xent(_ptr(logits), logits.stride(0), _ptr(node_labels), _ptr(nodes),
                                  _ptr(n_dev), dy.shape[0], int(num_classes), _ptr(dy),
                                  dy.stride(0), dy.shape[1], _ptr(loss), _ptr(row_loss),
                                  _ptr(status), _stream()))


def adam_step(w: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int,
              lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=5e-4):
    """NEXT-4 optimizer step (R34) on flat fp32 buffers, in place."""
    _check(lib().cmb_adam_step(_ptr(w), _ptr(g), _ptr(m), _ptr(v), w.numel(), lr, beta1, beta2,
                               eps, weight_decay, int(step), _stream()))


def _workspace(nbytes: int, device) -> torch.Tensor:
    # zero-initialised: its first word is the sticky device status (include/cmb.h)
    return torch.zeros(max(256, int(nbytes)), dtype=torch.uint8, device=device)


class Graph:
    """a0: a community-ordered CSR graph (+ optional feature table) resident in HBM."""

    def __init__(self, indptr, indices, community, num_communities, features=None, feat_dim=None,
                 validate=True, device="cuda"):
        dev = torch.device(device)
        self.device = dev
        self.indptr = _dev_tensor(indptr, torch.int64, dev)
        self.indices = _dev_tensor(indices, torch.int32, dev)
        self.community = _dev_tensor(community, torch.int32, dev)
        self.num_nodes = int(self.indptr.shape[0] - 1)
        self.num_edges = int(self.indices.shape[0])
        self.num_communities = int(num_communities)
        self.features = None
        self.feat_dim = 0
        self.feat_ld = 0
        if features is not None:
            X = features if isinstance(features, torch.Tensor) else torch.as_tensor(features)
            X = X.to(device=dev, dtype=torch.float32)
            if X.dim() != 2 or X.stride(1) != 1:
                X = X.contiguous()
            self.features = X
            self.feat_dim = int(feat_dim if feat_dim is not None else X.shape[1])
            self.feat_ld = int(X.stride(0))
        nb = lib().cmb_graph_workspace_bytes(self.num_nodes, self.num_communities)
        self.workspace = _workspace(nb, dev)
        d = GraphDesc(self.num_nodes, self.num_edges, self.indptr.data_ptr(),
                      self.indices.data_ptr(), self.community.data_ptr(), self.num_communities,
                      self.features.data_ptr() if self.features is not None else None,
                      self.feat_dim, self.feat_ld, self.workspace.data_ptr(), nb, int(validate))
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().cmb_load_graph(ctypes.byref(d), _stream(), ctypes.byref(h)))
        self.handle = h

    @classmethod
    def from_bundle(cls, bundle, device="cuda", features=True, validate=True):
        """features: True (the bundle's host table), False, or a ready [N, ld] tensor."""
        if isinstance(features, torch.Tensor):
            X = features
        else:
            X = torch.from_numpy(bundle.X) if (features and bundle.X is not None) else None
        return cls(torch.from_numpy(bundle.indptr), torch.from_numpy(bundle.indices),
                   torch.from_numpy(bundle.comm), bundle.cfg.num_communities, X,
                   bundle.cfg.feat_dim if X is not None else None, validate, device)

    def arrays(self):
        """(cbeg int32[C+1], bounds int32[N, 2]) device tensors produced by a0."""
        cb, bd = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().cmb_graph_arrays(self.handle, ctypes.byref(cb), ctypes.byref(bd)))
        ws = self.workspace
        base = ws.data_ptr()
        cbeg = ws[cb.value - base: cb.value - base + 4 * (self.num_communities + 1)].view(torch.int32)
        bounds = ws[bd.value - base: bd.value - base + 8 * self.num_nodes].view(torch.int32)
        return cbeg, bounds.view(self.num_nodes, 2)

    def status(self):
        return lib().cmb_get_device_status(_ptr(self.workspace), _stream())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.cmb_free_graph(h)
            self.handle = None


class RootOrderer:
    """a1: Knob-1 root order per epoch (owns its workspace)."""

    def __init__(self, graph: Graph, train):
        self.graph = graph
        self.train = _dev_tensor(train, torch.int32, graph.device)
        self.n = int(self.train.shape[0])
        self.workspace = _workspace(lib().cmb_order_roots_workspace_bytes(self.n,
                                                                          graph.num_communities),
                                    graph.device)
        self.out = torch.empty(self.n, dtype=torch.int32, device=graph.device)

    def order(self, mode="rand", mix=0.0, seed=42, epoch=0, out=None):
        m = _MODES[mode] if isinstance(mode, str) else int(mode)
        o = self.out if out is None else out
        _check(lib().cmb_order_roots(self.graph.handle, _ptr(self.train), self.n, m, float(mix),
                                     int(seed), int(epoch), _ptr(o), _ptr(self.workspace),
                                     self.workspace.numel(), _stream()))
        return o

    def status(self):
        return lib().cmb_get_device_status(_ptr(self.workspace), _stream())


def order_roots(graph: Graph, train, mode="rand", mix=0.0, seed=42, epoch=0):
    return RootOrderer(graph, train).order(mode, mix, seed, epoch).clone()


def blocks_capacity(n_roots: int, fanouts: Sequence[int], num_nodes: int):
    L = len(fanouts)
    f = (ctypes.c_int32 * L)(*fanouts)
    nc = (ctypes.c_int64 * (L + 1))()
    ec = (ctypes.c_int64 * L)()
    lib().cmb_blocks_capacity(n_roots, f, L, num_nodes, nc, ec)
    return list(nc), list(ec)


@dataclass
class BatchView:
    """Device views of one sampled batch (valid until the next sample() call)."""
    nodes: torch.Tensor           # [nodes_cap] (valid prefix n_L)
    sizes: torch.Tensor           # [2L+1] n_0..n_L, e_0..e_{L-1} (device)
    indptr: List[torch.Tensor]    # hop h: [n_cap[h]+1]
    indices: List[torch.Tensor]   # hop h: [e_cap[h]]
    new_src_mask: torch.Tensor

    def host_sizes(self):
        s = self.sizes.cpu().tolist()
        L = len(self.indptr)
        return s[: L + 1], s[L + 1:]


class Sampler:
    """a2+a3 (+ a4/a5): owns the workspace and the output blocks for batches of at
    most `max_roots` roots with the given hop-ordered fanouts."""

    def __init__(self, graph: Graph, max_roots: int, fanouts: Sequence[int]):
        self.graph = graph
        self.fanouts = [int(f) for f in fanouts]
        self.L = L = len(self.fanouts)
        if not (1 <= L <= MAX_HOPS) or any(f < 1 or f > MAX_FANOUT for f in self.fanouts):
            raise ValueError("fanouts: 1..8 hops, each in [1, 32]")
        self.max_roots = int(max_roots)
        dev = graph.device
        self.n_cap, self.e_cap = blocks_capacity(self.max_roots, self.fanouts, graph.num_nodes)
        self._f = (ctypes.c_int32 * L)(*self.fanouts)
        self.workspace = _workspace(lib().cmb_sample_workspace_bytes(self.max_roots, self._f, L,
                                                                     graph.num_nodes), dev)
        self.nodes = torch.empty(self.n_cap[L], dtype=torch.int32, device=dev)
        self.indptr = [torch.empty(self.n_cap[h] + 1, dtype=torch.int32, device=dev)
                       for h in range(L)]
        self.indices = [torch.empty(max(1, self.e_cap[h]), dtype=torch.int32, device=dev)
                        for h in range(L)]
        self.mask = torch.empty((self.e_cap[L - 1] + 31) // 32 + 1, dtype=torch.int32, device=dev)
        self.last_src_ids = torch.empty(max(1, self.e_cap[L - 1]), dtype=torch.int32, device=dev)
        self.sizes = torch.zeros(2 * L + 1, dtype=torch.int64, device=dev)
        b = Blocks()
        b.nodes = self.nodes.data_ptr()
        b.nodes_cap = self.n_cap[L]
        for h in range(L):
            b.indptr[h] = self.indptr[h].data_ptr()
            b.indices[h] = self.indices[h].data_ptr()
            b.indices_cap[h] = self.e_cap[h]
        b.new_src_mask = self.mask.data_ptr()
        b.last_src_ids = self.last_src_ids.data_ptr()
        b.sizes = self.sizes.data_ptr()
        # the visiting order of the last hop's dst rows, written by the sampler and used by the
        # a4 + a5 calls (include/cmb.h cmb_blocks.dst_order; results do not depend on it)
        self.dst_order = torch.empty(max(1, self.n_cap[L - 1]), dtype=torch.int32, device=dev)
        b.dst_order = self.dst_order.data_ptr()
        self._blocks = b
        self.x_in = None
        self.h = None

    def sample(self, roots: torch.Tensor, p: float, seed: int, batch_id: int,
               law=LAW_A) -> BatchView:
        n = int(roots.shape[0])
        if n > self.max_roots:
            raise ValueError("more roots than max_roots")
        lw = _law(law)
        if lw == LAW_A:
            _check(lib().cmb_sample_blocks(self.graph.handle, _ptr(roots), n, self._f, self.L,
                                           float(p), int(seed), int(batch_id),
                                           ctypes.byref(self._blocks), _ptr(self.workspace),
                                           self.workspace.numel(), _stream()))
        else:
            _check(lib().cmb_sample_blocks_law(self.graph.handle, _ptr(roots), n, self._f,
                                               self.L, float(p), lw, int(seed), int(batch_id),
                                               ctypes.byref(self._blocks), _ptr(self.workspace),
                                               self.workspace.numel(), _stream()))
        return BatchView(self.nodes, self.sizes, self.indptr, self.indices, self.mask)

    def batch_desc(self, roots: torch.Tensor, batch_id: int) -> "Batch":
        n = int(roots.shape[0])
        if n > self.max_roots:
            raise ValueError("more roots than max_roots")
        return Batch(roots.data_ptr(), n, int(batch_id), ctypes.pointer(self._blocks),
                     self.workspace.data_ptr(), self.workspace.numel())

    def alloc_features(self):
        g = self.graph
        if self.x_in is None:
            self.x_in = torch.empty(self.n_cap[self.L], g.feat_ld, dtype=torch.float32,
                                    device=g.device)
            self.h = torch.empty(self.n_cap[self.L - 1], g.feat_ld, dtype=torch.float32,
                                 device=g.device)
        return self.x_in, self.h

    def gather_aggregate(self):
        """a4 + a5 fused for the last sampled batch -> (X_in [n_L, ld], H [n_{L-1}, ld])."""
        x_in, h = self.alloc_features()
        _check(lib().cmb_gather_aggregate(self.graph.handle, ctypes.byref(self._blocks), self.L,
                                          self.n_cap[self.L - 1], self.n_cap[self.L], _ptr(x_in),
                                          x_in.stride(0), _ptr(h), h.stride(0), _stream()))
        return x_in, h

    def gather_aggregate_sharded(self, table: "ShardTable"):
        """NEXT-1: a4 + a5 reading every feature row from its owner's shard (peer shards mapped
        over NVLink); same bytes as gather_aggregate on the concatenated table."""
        x_in, h = self.alloc_features_ld(table.feat_ld)
        _check(lib().cmb_gather_aggregate_sharded(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            self.n_cap[self.L], table.ptr_array, table.world, table.rows_per_shard, table.shard_ld,
            table.feat_dim, _ptr(x_in), x_in.stride(0), _ptr(h), h.stride(0), _stream()))
        return x_in, h

    def gather_aggregate_cached(self, cache: "FeatureCache"):
        """NEXT-3: a4 + a5 through the HBM feature cache (misses read from the host table)."""
        x_in, h = self.alloc_features_ld(cache.rows.stride(0))
        _check(lib().cmb_cache_gather_aggregate(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            self.n_cap[self.L], ctypes.byref(cache.desc), cache.feat_dim, cache.next_tag(),
            _ptr(x_in), x_in.stride(0), _ptr(h), h.stride(0), _ptr(cache.stats), _stream()))
        return x_in, h

    def saved_a_buffer(self) -> torch.Tensor:
        """Device buffer for the layer-1 operand tiles saved by sage_layer(save_a=True)."""
        n = lib().cmb_sage_saved_a_bytes(self.graph.feat_dim, self.n_cap[self.L - 1])
        if getattr(self, "_a_save", None) is None or self._a_save.numel() < n:
            self._a_save = torch.empty(max(16, n), dtype=torch.uint8, device=self.graph.device)
        return self._a_save

    def sage_layer(self, layer: "SageLayer", out: Optional[torch.Tensor] = None,
                   save_a: bool = False):
        """NEXT-4: a4 + a5 fused with the first GraphSAGE layer for the last sampled batch ->
        Y [n_cap[L-1], out_dim] (rows < n_{L-1} valid), fp32 or bf16 as the layer says.
        save_a: also keep the operand tiles for sage_layer_backward(saved=True)."""
        if out is None:
            out = layer.alloc_out(self.n_cap[self.L - 1])
        if save_a:
            a = self.saved_a_buffer()
            _check(lib().cmb_sage_layer_forward_save(
                self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
                _ptr(layer.w_img), _ptr(layer.bias), layer.out_dim, int(layer.relu),
                int(layer.out_bf16), _ptr(out), out.stride(0), _ptr(a), a.numel(), _stream()))
            return out
        _check(lib().cmb_sage_layer_forward(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            _ptr(layer.w_img), _ptr(layer.bias), layer.out_dim, int(layer.relu),
            int(layer.out_bf16), _ptr(out), out.stride(0), _stream()))
        return out

    def sage_hidden(self, layer: "SageLayer", hop: int, y_prev: torch.Tensor,
                    out: Optional[torch.Tensor] = None):
        """NEXT-4 hidden layer (R29) on hop `hop` of the last sampled batch: y_prev = the
        previous layer's bf16 output (rows = local src ids of the hop) -> Y [n_cap[hop], out]."""
        if not layer.hidden:
            raise ValueError("layer was packed as a first layer; use SageLayer(..., hidden=True)")
        if y_prev.dtype != torch.bfloat16:
            raise ValueError("y_prev must be bf16")
        if out is None:
            out = layer.alloc_out(self.n_cap[hop])
        _check(lib().cmb_sage_hidden_forward(
            ctypes.byref(self._blocks), int(hop), self.n_cap[hop], _ptr(y_prev), y_prev.stride(0),
            layer.feat_dim, _ptr(layer.w_img), _ptr(layer.bias), layer.out_dim, int(layer.relu),
            int(layer.out_bf16), _ptr(out), out.stride(0), _stream()))
        return out

    def gcn_layer(self, layer: "GcnLayer", out: Optional[torch.Tensor] = None):
        """NEXT-4 GCN variant (R28): a4 + A' = (D + I)^-1 (A + I) aggregation + X W on tcgen05."""
        if out is None:
            out = layer.alloc_out(self.n_cap[self.L - 1])
        _check(lib().cmb_gcn_layer_forward(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            _ptr(layer.w_img), _ptr(layer.bias), layer.out_dim, int(layer.relu),
            int(layer.out_bf16), _ptr(out), out.stride(0), _stream()))
        return out

    def sage_dense_layer(self, layer: "DenseSageLayer", out: Optional[torch.Tensor] = None):
        """NEXT-4 for wide rows (F > 128): a4 + a5 (cmb_gather_aggregate) for the last sampled
        batch, then the layer on its X_in / H (cmb_sage_dense_forward) -> Y [n_cap[L-1], out]."""
        cap = self.n_cap[self.L - 1]
        if out is None:
            out = layer.alloc_out(cap)
        x_in, h = self.gather_aggregate()
        ws = layer.workspace(cap)
        _check(lib().cmb_sage_dense_forward(
            _ptr(x_in), x_in.stride(0), _ptr(h), h.stride(0), _ptr(self.sizes[self.L - 1:self.L]),
            cap, layer.feat_dim, _ptr(layer.w_img), _ptr(layer.bias), layer.out_dim,
            int(layer.relu), int(layer.out_bf16), _ptr(out), out.stride(0), _ptr(ws), ws.numel(),
            _stream()))
        return out

    def sage_dense_backward(self, layer: "DenseSageLayer", dy: torch.Tensor,
                            y: Optional[torch.Tensor] = None, dw: Optional[torch.Tensor] = None,
                            db: Optional[torch.Tensor] = None):
        """Weight gradients of sage_dense_layer on the X_in / H of the last gather (R27)."""
        if dy.dtype not in (torch.bfloat16, torch.float32) or (
                y is not None and y.dtype != torch.bfloat16):
            raise ValueError("dy must be bf16 or fp32, y bf16")
        F, fo = layer.feat_dim, layer.out_dim
        cap = self.n_cap[self.L - 1]
        dw, db = _grad_out(dw, db, F, fo, layer.device)
        ws = layer.workspace(cap)
        x_in, h = self.x_in, self.h
        _check(lib().cmb_sage_dense_backward(
            _ptr(x_in), x_in.stride(0), _ptr(h), h.stride(0), _ptr(self.sizes[self.L - 1:self.L]),
            cap, F, _ptr(dy), dy.stride(0), int(dy.dtype == torch.float32), _ptr(y),
            0 if y is None else y.stride(0), fo, _ptr(dw), _ptr(db), _ptr(ws), ws.numel(),
            _stream()))
        return dw[0], dw[1], db

    def gcn_layer_backward(self, layer: "GcnLayer", dy: torch.Tensor,
                           y: Optional[torch.Tensor] = None):
        """NEXT-4 GCN backward (R35) for the last sampled batch: dY (bf16 or fp32
        [>= n_{L-1}, out_dim]) and, for a ReLU layer, its bf16 output Y -> (dW [F, out], db)."""
        if dy.dtype not in (torch.bfloat16, torch.float32) or (
                y is not None and y.dtype != torch.bfloat16):
            raise ValueError("dy must be bf16 or fp32, y bf16")
        F, fo = layer.feat_dim, layer.out_dim
        ws = layer.backward_workspace()
        dw = torch.empty(F, fo, dtype=torch.float32, device=layer.device)
        db = torch.empty(fo, dtype=torch.float32, device=layer.device)
        _check(lib().cmb_gcn_layer_backward(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            _ptr(dy), dy.stride(0), int(dy.dtype == torch.float32), _ptr(y),
            0 if y is None else y.stride(0), fo, _ptr(dw), _ptr(db), _ptr(ws), ws.numel(),
            _stream()))
        return dw, db

    def sage_layer_backward(self, layer: "SageLayer", dy: torch.Tensor,
                            y: Optional[torch.Tensor] = None, dw: Optional[torch.Tensor] = None,
                            db: Optional[torch.Tensor] = None, saved: bool = False):
        """NEXT-4 backward for the last sampled batch: dY (bf16 [>= n_{L-1}, out_dim]) and, for a
        ReLU layer, its output Y (bf16) -> (dW_self [F, out_dim], dW_neigh, db) fp32."""
        if dy.dtype not in (torch.bfloat16, torch.float32) or (
                y is not None and y.dtype != torch.bfloat16):
            raise ValueError("dy must be bf16 or fp32, y bf16")
        F, fo = layer.feat_dim, layer.out_dim
        ws = layer.backward_workspace()
        dw, db = _grad_out(dw, db, F, fo, layer.device)
        if saved:   # the operand tiles of the last sage_layer(save_a=True) on this batch
            a = self.saved_a_buffer()
            _check(lib().cmb_sage_layer_backward_saved(
                self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
                _ptr(a), a.numel(), _ptr(dy), dy.stride(0), int(dy.dtype == torch.float32),
                _ptr(y), 0 if y is None else y.stride(0), fo, _ptr(dw), _ptr(db), _ptr(ws),
                ws.numel(), _stream()))
            return dw[0], dw[1], db
        _check(lib().cmb_sage_layer_backward(
            self.graph.handle, ctypes.byref(self._blocks), self.L, self.n_cap[self.L - 1],
            _ptr(dy), dy.stride(0), int(dy.dtype == torch.float32), _ptr(y),
            0 if y is None else y.stride(0), fo, _ptr(dw), _ptr(db), _ptr(ws), ws.numel(),
            _stream()))
        return dw[0], dw[1], db

    def sage_hidden_backward(self, layer: "SageLayer", hop: int, y_prev: torch.Tensor,
                             dy: torch.Tensor, y: Optional[torch.Tensor] = None,
                             dz_out: Optional[torch.Tensor] = None,
                             dw: Optional[torch.Tensor] = None, db: Optional[torch.Tensor] = None):
        """NEXT-4 hidden-layer backward (R31) on hop `hop` of the last sampled batch: y_prev =
        the layer's bf16 input (the previous layer's output), dY (bf16 [>= n_hop, out_dim]) and,
        for a ReLU layer, its output Y (bf16) -> (dW_self [F, out], dW_neigh, db) fp32.
        dz_out (bf16 [>= n_hop, >= out_dim]) receives the masked dZ for sage_hidden_input_grad."""
        if not layer.hidden:
            raise ValueError("layer was packed as a first layer; use SageLayer(..., hidden=True)")
        if any(t is not None and t.dtype != torch.bfloat16 for t in (y_prev, y)) or \
                dy.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("y_prev and y must be bf16, dy bf16 or fp32")
        F, fo = layer.feat_dim, layer.out_dim
        ws = layer.backward_workspace()
        dw, db = _grad_out(dw, db, F, fo, layer.device)
        _check(lib().cmb_sage_hidden_backward(
            ctypes.byref(self._blocks), int(hop), self.n_cap[hop], _ptr(y_prev), y_prev.stride(0),
            F, _ptr(dy), dy.stride(0), int(dy.dtype == torch.float32), _ptr(y),
            0 if y is None else y.stride(0), fo, _ptr(dw),
            _ptr(db), _ptr(ws), ws.numel(), _ptr(dz_out),
            0 if dz_out is None else dz_out.stride(0), _stream()))
        return dw[0], dw[1], db

    def sage_hidden_input_grad(self, layer: "SageLayer", hop: int, dz: torch.Tensor,
                               dx: Optional[torch.Tensor] = None):
        """NEXT-4 (R32): gradient into a hidden layer's input Yp from dZ (bf16 [>= n_hop, ld],
        ld >= out_dim rounded up to 64, padding columns zero) -> dX fp32 [n_cap[hop+1], in_dim]
        (rows >= n_{hop+1} zero)."""
        if not layer.hidden or dz.dtype != torch.bfloat16:
            raise ValueError("needs a hidden SageLayer and a bf16 dz")
        F, fo = layer.feat_dim, layer.out_dim
        wt = layer.transposed_image()
        if dx is None:
            dx = torch.empty(self.n_cap[hop + 1], F, dtype=torch.float32, device=layer.device)
        dh = torch.empty(max(1, self.n_cap[hop]), F, dtype=torch.float32, device=layer.device)
        _check(lib().cmb_sage_hidden_input_grad(
            ctypes.byref(self._blocks), int(hop), self.n_cap[hop], self.n_cap[hop + 1], _ptr(dz),
            dz.stride(0), fo, _ptr(wt), F, _ptr(dx), dx.stride(0), _ptr(dh), dh.stride(0),
            _stream()))
        return dx

    def alloc_features_ld(self, ld: int):
        if self.x_in is None or self.x_in.stride(0) != ld:
            dev = self.graph.device
            self.x_in = torch.empty(self.n_cap[self.L], ld, dtype=torch.float32, device=dev)
            self.h = torch.empty(self.n_cap[self.L - 1], ld, dtype=torch.float32, device=dev)
        return self.x_in, self.h

    def set_dst_order(self, enabled: bool):
        """Let the sampler write (and the a4 + a5 calls use) the dst visiting order, or not."""
        self._blocks.dst_order = self.dst_order.data_ptr() if enabled else None

    def status(self):
        return lib().cmb_get_device_status(_ptr(self.workspace), _stream())


class SageLayer:
    """NEXT-4 (R26): weights of the input-side SAGEConv-mean layer, packed once into the
    tensor cores' bf16 operand image.  w_self / w_neigh: [F, out_dim] (Y = X W), bias: [out_dim]."""

    def __init__(self, w_self: torch.Tensor, w_neigh: torch.Tensor, bias=None, relu=True,
                 out_bf16=False, device=None, hidden=False):
        F, fo = int(w_self.shape[0]), int(w_self.shape[1])
        if tuple(w_neigh.shape) != (F, fo):
            raise ValueError("w_self and w_neigh must both be [F, out_dim]")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.hidden = bool(hidden)  # packed for cmb_sage_hidden_forward (layers >= 2, R29)
        nbytes = (lib().cmb_sage_hidden_weights_bytes if hidden else lib().cmb_sage_weights_bytes)(F, fo)
        if nbytes == 0:
            raise ValueError(f"unsupported layer shape F={F}, out_dim={fo} (F <= 128, out_dim in "
                             f"[16, 256], a multiple of 16)")
        self.feat_dim, self.out_dim = F, fo
        self.relu, self.out_bf16 = bool(relu), bool(out_bf16)
        self.w_self = _dev_tensor(w_self, torch.float32, dev)
        self.w_neigh = _dev_tensor(w_neigh, torch.float32, dev)
        self.bias = None if bias is None else _dev_tensor(bias, torch.float32, dev)
        self.w_img = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.device = dev
        self.repack()

    def repack(self):
        self._wt = None  # the transposed image follows the weights
        pack = lib().cmb_sage_hidden_pack_weights if self.hidden else lib().cmb_sage_pack_weights
        _check(pack(_ptr(self.w_self), _ptr(self.w_neigh), self.feat_dim, self.out_dim,
                    _ptr(self.w_img), self.w_img.numel(), _stream()))

    def transposed_image(self) -> torch.Tensor:
        """bf16 image of (W_self^T, W_neigh^T) for the input-gradient GEMMs (R32); rebuilt by
        repack()."""
        if getattr(self, "_wt", None) is None:
            n = lib().cmb_sage_hidden_weights_t_bytes(self.feat_dim, self.out_dim)
            if n == 0:
                raise ValueError(f"input gradient needs in_dim in [16, 256] a multiple of 16 "
                                 f"(got {self.feat_dim})")
            self._wt = torch.empty(n, dtype=torch.uint8, device=self.device)
            _check(lib().cmb_sage_hidden_pack_weights_t(
                _ptr(self.w_self), _ptr(self.w_neigh), self.feat_dim, self.out_dim,
                _ptr(self._wt), self._wt.numel(), _stream()))
        return self._wt

    def backward_workspace(self) -> torch.Tensor:
        if getattr(self, "_bws", None) is None:
            n = (lib().cmb_sage_hidden_backward_workspace_bytes if self.hidden else
                 lib().cmb_sage_backward_workspace_bytes)(self.feat_dim, self.out_dim)
            if n == 0:
                raise ValueError(f"backward needs out_dim a power of two in [16, 256] "
                                 f"(got {self.out_dim})")
            self._bws = torch.empty(n, dtype=torch.uint8, device=self.device)
        return self._bws

    def alloc_out(self, rows: int) -> torch.Tensor:
        dt = torch.bfloat16 if self.out_bf16 else torch.float32
        return torch.empty(max(1, rows), self.out_dim, dtype=dt, device=self.device)


class DenseSageLayer:
    """NEXT-4 first layer for wide feature rows (F > 128, e.g. Reddit's 602; include/cmb.h
    cmb_sage_dense_*): the weights [F, out_dim] (Y = X W) packed once into a bf16 image; the
    layer runs on the a4 + a5 outputs of the fused gather."""

    def __init__(self, w_self: torch.Tensor, w_neigh: torch.Tensor, bias=None, relu=True,
                 out_bf16=False, device=None):
        F, fo = int(w_self.shape[0]), int(w_self.shape[1])
        if tuple(w_neigh.shape) != (F, fo):
            raise ValueError("w_self and w_neigh must both be [F, out_dim]")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = lib().cmb_sage_dense_weights_bytes(F, fo)
        if nbytes == 0:
            raise ValueError(f"unsupported dense layer shape F={F}, out_dim={fo}")
        self.feat_dim, self.out_dim = F, fo
        self.relu, self.out_bf16 = bool(relu), bool(out_bf16)
        self.hidden = False
        self.w_self = _dev_tensor(w_self, torch.float32, dev)
        self.w_neigh = _dev_tensor(w_neigh, torch.float32, dev)
        self.bias = None if bias is None else _dev_tensor(bias, torch.float32, dev)
        self.w_img = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self.device = dev
        self._ws = {}
        self.repack()

    def repack(self):
        _check(lib().cmb_sage_dense_pack_weights(_ptr(self.w_self), _ptr(self.w_neigh),
                                                 self.feat_dim, self.out_dim, _ptr(self.w_img),
                                                 self.w_img.numel(), _stream()))

    def workspace(self, rows_cap: int) -> torch.Tensor:
        ws = self._ws.get(rows_cap)
        if ws is None:
            n = lib().cmb_sage_dense_workspace_bytes(rows_cap, self.feat_dim, self.out_dim)
            ws = _workspace(n, self.device)
            self._ws[rows_cap] = ws
        return ws

    def alloc_out(self, rows: int) -> torch.Tensor:
        dt = torch.bfloat16 if self.out_bf16 else torch.float32
        return torch.empty(max(1, rows), self.out_dim, dtype=dt, device=self.device)


class GraphSAGE:
    """NEXT-4: the paper's L-layer GraphSAGE (3 layers, hidden 256, DGL defaults
    lr 1e-3, weight decay 5e-4) trained on the sampled blocks of a Sampler, every stage in this
    library's kernels: layer 1 fused with a4 + a5 (R26), hidden layers (R29), softmax
    cross-entropy (R33), weight gradients (R27, R31), input gradients of the hidden layers (R32),
    Adam (R34), weight images repacked.  All parameters live in ONE flat fp32 buffer (per layer
    [W_self | W_neigh | b]) with matching gradient and moment buffers, so the optimizer is one
    launch.  The last layer's width is num_classes rounded up to a power of two >= 16 (the padded
    columns start at zero and stay zero: no gradient reaches them)."""

    def __init__(self, feat_dim: int, num_classes: int, hidden: int = 256, num_layers: int = 3,
                 seed: int = 0, lr=1e-3, weight_decay=5e-4, device=None):
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        out = 16
        while out < num_classes:
            out *= 2
        self.dims = [feat_dim] + [hidden] * (num_layers - 1) + [out]
        self.num_classes, self.L = int(num_classes), num_layers
        self.lr, self.weight_decay, self.step_count = lr, weight_decay, 0
        sizes = [2 * self.dims[l] * self.dims[l + 1] + self.dims[l + 1] for l in range(num_layers)]
        self.offsets = [sum(sizes[:l]) for l in range(num_layers + 1)]
        n = self.offsets[-1]
        gen = torch.Generator().manual_seed(seed)
        host = torch.zeros(n)
        for l in range(num_layers):   # Glorot-uniform weights, zero bias (DGL's SAGEConv init)
            fi, fo = self.dims[l], self.dims[l + 1]
            a = (6.0 / (fi + fo)) ** 0.5
            w = (torch.rand(2, fi, fo, generator=gen) * 2 - 1) * a
            if l == num_layers - 1:
                w[:, :, num_classes:] = 0.0
            host[self.offsets[l]:self.offsets[l] + 2 * fi * fo] = w.reshape(-1)
        self.params = host.to(dev)
        self.grads = torch.zeros(n, device=dev)
        self.m = torch.zeros(n, device=dev)
        self.v = torch.zeros(n, device=dev)
        self.layers = []
        for l in range(num_layers):
            ws, wn, b = self._views(self.params, l)
            last = l == num_layers - 1
            if l == 0 and feat_dim > 128:  # wide rows: the unfused dense first layer
                self.layers.append(DenseSageLayer(ws, wn, b, relu=not last, out_bf16=not last,
                                                  device=dev))
                continue
            self.layers.append(SageLayer(ws, wn, b, relu=not last, out_bf16=not last,
                                         device=dev, hidden=l > 0))
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self._bufs = {}
        self._step_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # graph-replayed steps
        self._step_synced = 0  # step_count the device counter matched when last written
        self._graphs = {}
        self.device = dev
        # layer 1's operand tiles are saved by the forward and reloaded by the backward instead
        # of re-gathering the feature rows; False re-gathers (same results)
        self.save_a = True

    def _views(self, flat, l):
        fi, fo = self.dims[l], self.dims[l + 1]
        o = self.offsets[l]
        return (flat[o:o + fi * fo].view(fi, fo), flat[o + fi * fo:o + 2 * fi * fo].view(fi, fo),
                flat[o + 2 * fi * fo:o + 2 * fi * fo + fo])

    def _buf(self, key, rows, cols, dtype):
        t = self._bufs.get(key)
        if t is None or t.shape[0] < rows:
            t = torch.zeros(max(1, rows), cols, dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def forward(self, sampler: "Sampler"):
        """Activations of every layer for the last sampled batch: [Y1, .., YL] (YL = fp32
        logits [n_cap[0], out], the others bf16)."""
        L = self.L
        if sampler.L != L:
            raise ValueError(f"sampler has {sampler.L} hops, the model {L} layers")
        ys = []
        for l, layer in enumerate(self.layers):
            h = L - 1 - l
            out = self._buf(("y", l), sampler.n_cap[h], layer.out_dim,
                            torch.bfloat16 if layer.out_bf16 else torch.float32)
            if l == 0 and isinstance(layer, DenseSageLayer):
                ys.append(sampler.sage_dense_layer(layer, out))
                continue
            ys.append(sampler.sage_layer(layer, out, save_a=self.save_a) if l == 0 else
                      sampler.sage_hidden(layer, h, ys[-1], out))
        return ys

    def train_step(self, sampler: "Sampler", node_labels: torch.Tensor,
                   graph: bool = False) -> torch.Tensor:
        """One training step on the last sampled batch: forward, loss, backward, Adam, repack.
        Returns the device fp64 loss tensor (no host synchronisation).

        graph=True: the step's ~20 launches are captured once per (sampler, labels) pair into a
        CUDA graph and replayed (no per-launch host cost or launch gaps).  Every launch reads its
        sizes from the device and the Adam step number from a device counter
        (cmb_adam_step_pack_dev), so a replay is exactly the eager step on the sampler's current
        batch.  The first call with a new pair runs the step eagerly (it sizes every buffer) and
        captures it for the next calls."""
        if not graph:
            return self._train_step(sampler, node_labels, dev_step=False)
        key = (id(sampler), node_labels.data_ptr())
        g = self._graphs.get(key)
        if g is not None:
            if int(self._step_synced) != self.step_count:  # eager host-step calls in between
                self._step_dev.fill_(self.step_count)
            g.replay()
            self.step_count += 1
            self._step_synced = self.step_count
            return self.loss
        self._train_step(sampler, node_labels, dev_step=True)       # eager: buffers sized
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self._train_step(sampler, node_labels, dev_step=True, count=False)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self._graphs[key] = g
        self._step_synced = self.step_count
        return self.loss

    def _train_step(self, sampler: "Sampler", node_labels: torch.Tensor, dev_step: bool,
                    count: bool = True) -> torch.Tensor:
        L = self.L
        ys = self.forward(sampler)
        fo = self.dims[-1]
        dy = self._buf("dyL", sampler.n_cap[0], fo, torch.bfloat16)
        softmax_xent(ys[-1], node_labels, sampler.nodes, sampler.sizes[0:1], self.num_classes,
                     dy[:sampler.n_cap[0]], self.loss, self.status,
                     self._buf("row_loss", sampler.n_cap[0], 1, torch.float64)[:, 0])
        for l in range(L - 1, -1, -1):
            h = L - 1 - l
            layer = self.layers[l]
            g_ws, g_wn, g_b = self._views(self.grads, l)
            dw = self.grads[self.offsets[l]:self.offsets[l] + 2 * g_ws.numel()].view(2, *g_ws.shape)
            y = ys[l] if layer.relu else None
            if l == 0 and isinstance(layer, DenseSageLayer):
                sampler.sage_dense_backward(layer, dy, y, dw=dw, db=g_b)
            elif l == 0:
                sampler.sage_layer_backward(layer, dy, y, dw=dw, db=g_b, saved=self.save_a)
            else:
                dz = self._buf(("dz", l), sampler.n_cap[h], ((layer.out_dim + 63) // 64) * 64,
                               torch.bfloat16)
                sampler.sage_hidden_backward(layer, h, ys[l - 1], dy, y, dz_out=dz, dw=dw, db=g_b)
                dy = sampler.sage_hidden_input_grad(
                    layer, h, dz, self._buf(("dx", l), sampler.n_cap[h + 1], layer.feat_dim,
                                            torch.float32)[:sampler.n_cap[h + 1]])
        if count:
            self.step_count += 1
        # Adam and the repack of every weight image (forward and transposed) in one launch
        packs = (LayerPack * L)()
        for l, layer in enumerate(self.layers):
            wt = layer.transposed_image() if layer.hidden else None
            packs[l] = LayerPack(self.offsets[l], layer.feat_dim, layer.out_dim,
                                 layer.w_img.data_ptr(), None if wt is None else wt.data_ptr(),
                                 int(isinstance(layer, DenseSageLayer)))
        if dev_step:  # the device counter holds the steps taken so far (eager or replayed)
            if count:
                self._step_dev.fill_(self.step_count - 1)
            _check(lib().cmb_adam_step_pack_dev(
                _ptr(self.params), _ptr(self.grads), _ptr(self.m), _ptr(self.v),
                self.params.numel(), self.lr, 0.9, 0.999, 1e-8, self.weight_decay,
                _ptr(self._step_dev), packs, L, _stream()))
        else:
            _check(lib().cmb_adam_step_pack(
                _ptr(self.params), _ptr(self.grads), _ptr(self.m), _ptr(self.v),
                self.params.numel(), self.lr, 0.9, 0.999, 1e-8, self.weight_decay,
                self.step_count, packs, L, _stream()))
        return self.loss


class GcnLayer:
    """NEXT-4 GCN variant (R28): one weight matrix w [F, out_dim], packed once."""

    def __init__(self, w: torch.Tensor, bias=None, relu=True, out_bf16=False, device=None):
        F, fo = int(w.shape[0]), int(w.shape[1])
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = lib().cmb_gcn_weights_bytes(F, fo)
        if nbytes == 0:
            raise ValueError(f"unsupported layer shape F={F}, out_dim={fo}")
        self.feat_dim, self.out_dim = F, fo
        self.relu, self.out_bf16 = bool(relu), bool(out_bf16)
        self.w = _dev_tensor(w, torch.float32, dev)
        self.bias = None if bias is None else _dev_tensor(bias, torch.float32, dev)
        self.w_img = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.device = dev
        _check(lib().cmb_gcn_pack_weights(_ptr(self.w), F, fo, _ptr(self.w_img), nbytes,
                                          _stream()))

    def alloc_out(self, rows: int) -> torch.Tensor:
        dt = torch.bfloat16 if self.out_bf16 else torch.float32
        return torch.empty(max(1, rows), self.out_dim, dtype=dt, device=self.device)

    def backward_workspace(self) -> torch.Tensor:
        if getattr(self, "_bws", None) is None:
            n = lib().cmb_sage_backward_workspace_bytes(self.feat_dim, self.out_dim)
            if n == 0:
                raise ValueError(f"backward needs out_dim a power of two in [16, 256] "
                                 f"(got {self.out_dim})")
            self._bws = torch.empty(n, dtype=torch.uint8, device=self.device)
        return self._bws


class FeatureCache:
    """NEXT-3: `capacity` feature rows cached in HBM in front of a host-resident table (pinned,
    read by the device over the host link on a miss); CLOCK replacement."""

    def __init__(self, graph: Graph, host_x: torch.Tensor, feat_dim: int, capacity: int,
                 max_rows: int, max_edges: int):
        if host_x.device.type != "cpu" or not host_x.is_pinned():
            raise ValueError("host_x must be a pinned host tensor")
        if host_x.stride(1) != 1:
            raise ValueError("host_x rows must be contiguous")
        self.graph, self.host_x, self.feat_dim = graph, host_x, int(feat_dim)
        self.capacity, self.max_rows, self.max_edges = int(capacity), int(max_rows), int(max_edges)
        ld = (self.feat_dim + 3) // 4 * 4
        dev = graph.device
        nb = lib().cmb_feature_cache_bytes(graph.num_nodes, self.capacity, self.max_rows,
                                           self.max_edges)
        self.workspace = _workspace(nb, dev)
        self.rows = torch.empty(self.capacity, ld, dtype=torch.float32, device=dev)
        self.stats = torch.zeros(2, dtype=torch.int64, device=dev)  # rows, misses
        self.desc = FeatureCacheDesc(self.workspace.data_ptr(), self.workspace.numel(),
                                     graph.num_nodes, self.capacity, self.max_rows,
                                     self.max_edges, host_x.data_ptr(), host_x.stride(0),
                                     self.rows.data_ptr(), ld)
        self.tag = 0
        self.reset()

    def reset(self):
        _check(lib().cmb_feature_cache_init(self.workspace.data_ptr(), self.workspace.numel(),
                                            self.graph.num_nodes, self.capacity, self.max_rows,
                                            self.max_edges, _stream()))
        self.stats.zero_()

    def next_tag(self) -> int:
        self.tag = (self.tag + 1) % 0xFFFFFFFF
        return self.tag

    def miss_rate(self) -> float:
        r, m = self.stats.tolist()
        return m / r if r else 0.0


class ShardTable:
    """NEXT-1: the row-sharded feature table as seen by one process -- `world` device pointers,
    shard r holding rows [r*S, (r+1)*S).  Built from local tensors (virtual shards on one GPU,
    or world = 1) or by `ShardTable.exchange` (CUDA IPC handles shared over a process group,
    peers' shards mapped into this process)."""

    def __init__(self, shards: Sequence, num_nodes: int, feat_dim: int, shard_ld=None,
                 mapped_bases=()):
        """shards: per rank a device tensor [rows, ld] or a raw device pointer (int)."""
        self.world = len(shards)
        if not 1 <= self.world <= 8:
            raise ValueError("1..8 shards")
        self.rows_per_shard = (int(num_nodes) + self.world - 1) // self.world
        self.feat_dim = int(feat_dim)
        lds = {int(t.stride(0)) for t in shards if isinstance(t, torch.Tensor)}
        if shard_ld is not None:
            lds.add(int(shard_ld))
        if len(lds) != 1:
            raise ValueError("shards must share one row stride")
        self.shard_ld = self.feat_ld = lds.pop()
        self._keep = [t for t in shards if isinstance(t, torch.Tensor)]
        self._ptrs = [t.data_ptr() if isinstance(t, torch.Tensor) else int(t) for t in shards]
        self.ptr_array = (ctypes.c_void_p * self.world)(*self._ptrs)
        self._mapped = list(mapped_bases)

    @classmethod
    def exchange(cls, x_local: torch.Tensor, num_nodes: int, feat_dim: int, rank: int, world: int,
                 group=None):
        """Collective: every rank exports its shard, all-gathers the handles and maps the
        peers' shards (CUDA IPC; NVLink on a multi-GPU node).

        Ownership: the producer's stream is synchronised before the handle is published, so a
        peer never maps a shard whose fill is still pending; every rank must keep its shard
        allocated and unchanged until ``close()`` (a collective: it unmaps the peers' shards and
        then waits at a barrier, so no rank returns from it while a peer may still read)."""
        import torch.distributed as tdist
        torch.cuda.current_stream(x_local.device).synchronize()  # the shard's bytes are final
        h = (ctypes.c_char * 64)()
        off = ctypes.c_uint64()
        _check(lib().cmb_ipc_export(ctypes.c_void_p(x_local.data_ptr()), h, ctypes.byref(off)))
        mine = (bytes(h), int(off.value), int(x_local.stride(0)))
        allh = [None] * world
        tdist.all_gather_object(allh, mine, group=group)
        ptrs, bases = [], []
        for r, (hb, o, ld) in enumerate(allh):
            if ld != x_local.stride(0):
                raise ValueError("all shards must share one row stride")
            if r == rank:
                ptrs.append(x_local)
                continue
            p, b = ctypes.c_void_p(), ctypes.c_void_p()
            _check(lib().cmb_ipc_open((ctypes.c_char * 64).from_buffer_copy(hb), o,
                                      ctypes.byref(p), ctypes.byref(b)))
            ptrs.append(int(p.value))
            bases.append(int(b.value))
        t = cls(ptrs, num_nodes, feat_dim, shard_ld=x_local.stride(0), mapped_bases=bases)
        t._group, t._collective = group, True
        return t

    def close(self):
        """Unmap the peers' shards.  For a table built by ``exchange`` this is a collective:
        the device work reading the shards is finished first, then all ranks meet at a barrier,
        after which each owner may free or overwrite its own shard."""
        if self._mapped or getattr(self, "_collective", False):
            torch.cuda.synchronize()
        for b in self._mapped:
            _check(lib().cmb_ipc_close(ctypes.c_void_p(b)))
        self._mapped = []
        if getattr(self, "_collective", False):
            import torch.distributed as tdist
            tdist.barrier(group=self._group)
            self._collective = False


def sample_multi(samplers: Sequence["Sampler"], roots: Sequence[torch.Tensor],
                 batch_ids: Sequence[int], p: float, seed: int, law=LAW_A):
    """a2+a3 for up to 4 independent batches in ONE launch (cmb_sample_blocks_multi); the
    samplers must share graph and fanouts and own distinct workspaces."""
    s0 = samplers[0]
    n = len(samplers)
    if not (1 <= n <= MAX_BATCHES_PER_LAUNCH) or len(roots) != n or len(batch_ids) != n:
        raise ValueError("1..4 samplers, one roots tensor and batch id each")
    arr = (Batch * n)(*[s.batch_desc(r, b) for s, r, b in zip(samplers, roots, batch_ids)])
    _check(lib().cmb_sample_blocks_multi(s0.graph.handle, arr, n, s0._f, s0.L, float(p),
                                         _law(law), int(seed), _stream()))
    return [BatchView(s.nodes, s.sizes, s.indptr, s.indices, s.mask) for s in samplers]


def community_order(indptr, indices, community, num_communities: int, device="cuda"):
    """NEXT-2 (iii): community-ordered relabelling of an arbitrary graph on the GPU ->
    (perm new->old, inv old->new, indptr, indices, community) device tensors (reading R25)."""
    dev = torch.device(device)
    ip = _dev_tensor(indptr, torch.int64, dev)
    ix = _dev_tensor(indices, torch.int32, dev)
    cm = _dev_tensor(community, torch.int32, dev)
    n, nnz = int(ip.shape[0] - 1), int(ix.shape[0])
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    inv = torch.empty(n, dtype=torch.int32, device=dev)
    ip2 = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ix2 = torch.empty(max(1, nnz), dtype=torch.int32, device=dev)
    cm2 = torch.empty(n, dtype=torch.int32, device=dev)
    ws = _workspace(lib().cmb_community_order_workspace_bytes(n, nnz), dev)
    _check(lib().cmb_community_order(_ptr(ip), _ptr(ix), _ptr(cm), n, nnz, int(num_communities),
                                     _ptr(perm), _ptr(inv), _ptr(ip2), _ptr(ix2), _ptr(cm2),
                                     _ptr(ws), ws.numel(), _stream()))
    return perm, inv, ip2, ix2[:nnz], cm2


def gather_features(graph: Graph, node_ids: torch.Tensor, n_dev: torch.Tensor, out: torch.Tensor):
    """a4: out[i] = X[node_ids[i]] for i < n_dev[0] (n_dev: device int64 scalar tensor)."""
    _check(lib().cmb_gather_features(graph.handle, _ptr(node_ids), _ptr(n_dev), out.shape[0],
                                     _ptr(out), out.stride(0), _stream()))
    return out


def sage_mean_aggregate(indptr: torch.Tensor, indices: torch.Tensor, n_dst_dev: torch.Tensor,
                        src: torch.Tensor, feat_dim: int, out: torch.Tensor,
                        src_map: Optional[torch.Tensor] = None, n_dst_cap: Optional[int] = None):
    """a5: out[d] = mean over the CSR row d of src[row] (row = src_map[idx] if given)."""
    cap = out.shape[0] if n_dst_cap is None else n_dst_cap
    _check(lib().cmb_sage_mean_aggregate(_ptr(indptr), _ptr(indices), _ptr(n_dst_dev), cap,
                                         _ptr(src), src.stride(0), _ptr(src_map), int(feat_dim),
                                         _ptr(out), out.stride(0), _stream()))
    return out


class MiniBatchPipeline:
    """One COMM-RAND mini-batch step per call (Alg. 1), all on the GPU:
    Knob-1 order once per epoch, then per batch Knob-2 sampling + relabel (a2, a3) and
    the fused input-feature gather + SAGE-mean aggregation (a4, a5)."""

    def __init__(self, graph: Graph, train, batch_size: int, fanouts: Sequence[int],
                 mode="rand", mix=0.0, p=0.5, seed=42, law=LAW_A):
        self.graph = graph
        self.law = _law(law)
        self.orderer = RootOrderer(graph, train)
        self.batch_size = int(batch_size)
        self.n_batches = (self.orderer.n + self.batch_size - 1) // self.batch_size
        self.sampler = Sampler(graph, self.batch_size, fanouts)
        self.mode, self.mix, self.p, self.seed = mode, float(mix), float(p), int(seed)
        self.epoch = None
        self.order = None

    def start_epoch(self, epoch: int):
        self.order = self.orderer.order(self.mode, self.mix, self.seed, epoch)
        self.epoch = int(epoch)

    def batch_roots(self, b: int) -> torch.Tensor:
        return self.order[b * self.batch_size: min((b + 1) * self.batch_size, self.orderer.n)]

    def step(self, global_batch: int, roots: Optional[torch.Tensor] = None):
        """Run batch `global_batch` (= epoch * n_batches + b).  Returns (BatchView, X_in, H)."""
        epoch, b = divmod(int(global_batch), self.n_batches)
        if roots is None:
            if self.epoch != epoch:
                self.start_epoch(epoch)
            roots = self.batch_roots(b)
        view = self.sampler.sample(roots, self.p, self.seed, int(global_batch), self.law)
        x_in, h = self.sampler.gather_aggregate()
        return view, x_in, h


class BatchedPipeline(MiniBatchPipeline):
    """The same step, `nb` batches per sampler launch (cmb_sample_blocks_multi: the SMs are
    split between the batches so the latency-bound sampling phases overlap), followed by the
    fused gather + aggregate of each batch.  Same bytes as the sequential pipeline."""

    def __init__(self, graph: Graph, train, batch_size: int, fanouts: Sequence[int],
                 mode="rand", mix=0.0, p=0.5, seed=42, nb: int = 2, law=LAW_A):
        super().__init__(graph, train, batch_size, fanouts, mode, mix, p, seed, law)
        self.nb = int(nb)
        if not 1 <= self.nb <= MAX_BATCHES_PER_LAUNCH:
            raise ValueError(f"nb must be in [1, {MAX_BATCHES_PER_LAUNCH}]")
        self.samplers = [self.sampler] + [Sampler(graph, self.batch_size, fanouts)
                                          for _ in range(self.nb - 1)]
        # the samplers' size vectors as rows of one tensor: a group's sizes are one copy away
        L = self.sampler.L
        self.group_sizes = torch.zeros(self.nb, 2 * L + 1, dtype=torch.int64, device=graph.device)
        for i, s in enumerate(self.samplers):
            s.sizes = self.group_sizes[i]
            s._blocks.sizes = s.sizes.data_ptr()
        # step-executor argument arrays, filled once (per group only roots / ids change)
        self._batches = (Batch * self.nb)()
        self._feats = (BatchFeatures * self.nb)()
        for i, s in enumerate(self.samplers):
            x_in, h = s.alloc_features()
            self._batches[i] = Batch(0, 0, 0, ctypes.pointer(s._blocks), s.workspace.data_ptr(),
                                     s.workspace.numel())
            self._feats[i] = BatchFeatures(x_in.data_ptr(), x_in.stride(0), h.data_ptr(),
                                           h.stride(0), s.n_cap[s.L - 1], s.n_cap[s.L])

    def make_events(self, n: int = None):
        """2 + 2n timing events for one step_group call, created and recorded once (so their
        handles exist) -- preallocate them outside a timed region."""
        n = self.nb if n is None else n
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 + 2 * n)]
        for e in evs:
            e.record()
        return evs

    def step_group(self, gbs: Sequence[int], roots: Optional[Sequence[torch.Tensor]] = None,
                   events=None, sizes_out: Optional[torch.Tensor] = None):
        """Run the global batches `gbs` (at most nb) with one sampler launch, then the fused
        gather + aggregate of each.  `roots` optionally overrides the epoch order; `sizes_out`
        (int64 [>= n, 2L+1], device) receives the batches' size vectors instead of group_sizes
        (no copy kernel per group).  If `events`
        is a dict, ('sample' -> (start, end)) and ('gather' -> [(start, end), ...]) CUDA events
        are recorded around the launches.  Returns the samplers used (one per batch)."""
        gbs = [int(x) for x in gbs]
        if not 1 <= len(gbs) <= self.nb:
            raise ValueError(f"1..{self.nb} batches per group")
        if roots is None:
            roots = []
            for gb in gbs:
                epoch, b = divmod(gb, self.n_batches)
                if self.epoch != epoch:
                    if roots:  # epoch boundary inside the group: keep the earlier epoch's roots
                        roots = [r.clone() for r in roots]
                    self.start_epoch(epoch)
                roots.append(self.batch_roots(b))
        ss = self.samplers[: len(gbs)]
        n = len(gbs)
        ev_list = None
        if isinstance(events, dict):  # fresh events (convenient, but costs host time per group)
            ev_list = [torch.cuda.Event(enable_timing=True) for _ in range(2 + 2 * n)]
            for e in ev_list:  # materialise the cudaEvent_t handles
                e.record()
            events["sample"] = (ev_list[0], ev_list[1])
            events["gather"] = [(ev_list[2 + 2 * i], ev_list[3 + 2 * i]) for i in range(n)]
        elif events is not None:      # a pre-created list of 2 + 2n recorded-once events
            ev_list = events
        for i, (s, r, gb) in enumerate(zip(ss, roots, gbs)):
            nr = int(r.shape[0])
            if nr > s.max_roots:
                raise ValueError("more roots than max_roots")
            bt = self._batches[i]
            bt.roots, bt.n_roots, bt.batch_id = r.data_ptr(), nr, gb
            x_in, h = s.alloc_features()
            if self._feats[i].x_in != x_in.data_ptr():  # outputs were re-allocated
                self._feats[i] = BatchFeatures(x_in.data_ptr(), x_in.stride(0), h.data_ptr(),
                                               h.stride(0), s.n_cap[s.L - 1], s.n_cap[s.L])
        evp = None
        if ev_list is not None:
            evp = (ctypes.c_void_p * (2 + 2 * n))(*[e.cuda_event for e in ev_list[: 2 + 2 * n]])
        s0 = ss[0]
        if sizes_out is not None:  # this group's size vectors straight into the caller's rows
            if (sizes_out.dtype != torch.int64 or sizes_out.shape[0] < n or
                    sizes_out.shape[1] != 2 * s0.L + 1 or not sizes_out.is_contiguous()):
                raise ValueError("sizes_out: contiguous int64 [>= n, 2L+1]")
            for i, s in enumerate(ss):
                s._blocks.sizes = sizes_out[i].data_ptr()
        try:
            _check(lib().cmb_step_group(self.graph.handle, self._batches, self._feats, n, s0._f,
                                        s0.L, float(self.p), self.law, int(self.seed), evp,
                                        _stream()))
        finally:  # the launches captured the pointers; later calls use group_sizes again
            if sizes_out is not None:
                for s in ss:
                    s._blocks.sizes = s.sizes.data_ptr()
        return ss


class OverlappedPipeline(MiniBatchPipeline):
    """The same step with `depth` batches in flight: the sampler of batch k+1 (latency-bound,
    stream `s_sample`) runs while the fused gather + aggregate of batch k (HBM-bound, stream
    `s_gather`) streams features.  Outputs are `depth`-buffered; events order the reuse."""

    def __init__(self, graph: Graph, train, batch_size: int, fanouts: Sequence[int],
                 mode="rand", mix=0.0, p=0.5, seed=42, depth: int = 2, law=LAW_A):
        super().__init__(graph, train, batch_size, fanouts, mode, mix, p, seed, law)
        self.depth = int(depth)
        self.samplers = [self.sampler] + [Sampler(graph, self.batch_size, fanouts)
                                          for _ in range(self.depth - 1)]
        self.s_sample = torch.cuda.Stream(device=graph.device)
        self.s_gather = torch.cuda.Stream(device=graph.device)
        self.ev_sampled = [torch.cuda.Event() for _ in range(self.depth)]
        self.ev_gathered = [torch.cuda.Event() for _ in range(self.depth)]
        self.gather_events = None  # optional list collecting (start, end) events per gather

    def step(self, global_batch: int, roots: Optional[torch.Tensor] = None):
        """Enqueue batch `global_batch`; returns its Sampler (outputs valid once
        `ev_gathered[j]` completes, j = global_batch % depth).  Never blocks the host."""
        gb = int(global_batch)
        j = gb % self.depth
        s = self.samplers[j]
        epoch, b = divmod(gb, self.n_batches)
        with torch.cuda.stream(self.s_sample):
            self.s_sample.wait_event(self.ev_gathered[j])  # buffer j consumed by batch gb-depth
            if roots is None:
                if self.epoch != epoch:
                    self.start_epoch(epoch)
                roots = self.batch_roots(b)
            s.sample(roots, self.p, self.seed, gb, self.law)
            self.ev_sampled[j].record(self.s_sample)
        with torch.cuda.stream(self.s_gather):
            self.s_gather.wait_event(self.ev_sampled[j])
            if self.gather_events is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.s_gather)
            s.gather_aggregate()
            if self.gather_events is not None:
                e1.record(self.s_gather)
                self.gather_events.append((e0, e1))
            self.ev_gathered[j].record(self.s_gather)
        return s

    def join(self, stream=None):
        """Make `stream` (default: current) wait for all enqueued work."""
        st = stream if stream is not None else torch.cuda.current_stream()
        st.wait_stream(self.s_sample)
        st.wait_stream(self.s_gather)
