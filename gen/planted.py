"""Planted-community graph generator (input recipe).

Graphs are generated ALREADY community-ordered (the paper assumes community-
ordered inputs): community c owns node ids [cbeg[c], cend[c]).

* ``kind="sbm"``: plain stochastic block model (SPEC.md gen_sbm S:61-69).
* ``kind="dcsbm"``: degree-corrected planted partition (Chung-Lu inside and
  across communities): community sizes follow a truncated power law
  (beta = 1.5), node weights theta a truncated power law (gamma = 2.5); every
  node emits ~theta_v * d/(2 E[theta]) stubs, each stub lands in its own
  community with probability 1 - mu (target proportional to theta), else
  anywhere in the graph (proportional to theta).  The stub list is then
  symmetrised, self-loops dropped, duplicates removed and rows sorted, and
  the stub scale is re-tuned until the realised CSR nnz is within 2 % of the
  target (the realised value is recorded in ``Bundle.meta``).

Features: X[v, j] = k * 2^-23 - 1 with k uniform in [0, 2^24): exactly
representable fp32 values in [-1, 1).  Train set: ``n_train`` distinct nodes
drawn uniformly, ascending.

All randomness comes from numpy PCG64 generators keyed by (gen_seed, stream)
and the splitmix64 streams of gen_core.c keyed by (gen_seed, node);
no code here is shared with or imported by either implementation's
arithmetic.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field, asdict
from typing import Optional

import numpy as np

from .configs import GraphConfig

GEN_VERSION = 4


@dataclass
class Bundle:
    cfg: GraphConfig
    indptr: np.ndarray      # int64 [N+1]
    indices: np.ndarray     # int32 [nnz], strictly ascending per row
    comm: np.ndarray        # int32 [N], non-decreasing
    train: np.ndarray       # int32 [n_train], ascending unique
    X: Optional[np.ndarray] = None  # float32 [N, ld] (pad columns zero)
    meta: dict = field(default_factory=dict)

    @property
    def num_nodes(self) -> int:
        return int(self.indptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed, stream]))


def _power_law(rng, n, lo, hi, expo):
    """Inverse-CDF draws from p(x) ~ x^-expo on [lo, hi]."""
    u = rng.random(n)
    a = 1.0 - expo
    return (lo ** a + u * (hi ** a - lo ** a)) ** (1.0 / a)


def _community_sizes(cfg: GraphConfig, rng) -> np.ndarray:
    n, c = cfg.num_nodes, cfg.num_communities
    lo, hi = cfg.comm_size_range
    if lo == hi:
        s = np.full(c, lo, dtype=np.int64)
    else:
        s = _power_law(rng, c, float(lo), float(hi), 1.5)
        s = np.maximum(1, np.floor(s / s.sum() * n)).astype(np.int64)
    diff = n - int(s.sum())
    order = np.argsort(-s, kind="stable")
    i = 0
    while diff != 0:  # spread the rounding remainder over the largest communities
        j = order[i % c]
        step = 1 if diff > 0 else -1
        if s[j] + step >= 1:
            s[j] += step
            diff -= step
        i += 1
    return s


def _csr_from_keys(keys: np.ndarray, n: int):
    keys = np.unique(keys)
    src = (keys // n).astype(np.int64)
    dst = (keys % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    return indptr, dst


def _sbm(cfg: GraphConfig, comm: np.ndarray, rng):
    n = cfg.num_nodes
    size = cfg.comm_size_range[0]
    exp_deg = cfg.nnz_target / n
    p_in = exp_deg * (1 - cfg.mu) / (size - 1)
    p_out = exp_deg * cfg.mu / (n - size)
    iu, ju = np.triu_indices(n, k=1)
    prob = np.where(comm[iu] == comm[ju], p_in, p_out)
    keep = rng.random(iu.shape[0]) < prob
    a, b = iu[keep].astype(np.int64), ju[keep].astype(np.int64)
    keys = np.concatenate([a * n + b, b * n + a])
    return _csr_from_keys(keys, n)


_LIB = None


def _lib():
    """gen_core.c compiled on first use (also done by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        import ctypes
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "libgen_core.so")
        src = os.path.join(here, "gen_core.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", so + ".tmp", src])
            os.replace(so + ".tmp", so)
        lib = ctypes.CDLL(so)
        P = ctypes.c_void_p
        lib.gen_dcsbm.argtypes = [ctypes.c_int64, ctypes.c_int32, P, P, P, P, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_uint64, P, P, P]
        lib.gen_dcsbm.restype = ctypes.c_int
        lib.gen_free.argtypes = [P]
        _LIB = lib
    return _LIB


def _dcsbm_once(cfg, comm, cbeg, theta, cum, scale, seed):
    import ctypes
    lib = _lib()
    ip, ix, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.gen_dcsbm(cfg.num_nodes, cfg.num_communities, cbeg.ctypes.data, comm.ctypes.data,
                       theta.ctypes.data, cum.ctypes.data, float(cfg.mu), float(scale),
                       int(seed) & ((1 << 64) - 1), ctypes.byref(ip), ctypes.byref(ix), ctypes.byref(nnz))
    if rc != 0:
        raise MemoryError("gen_dcsbm failed")
    n = cfg.num_nodes
    indptr = np.ctypeslib.as_array((ctypes.c_int64 * (n + 1)).from_address(ip.value)).copy()
    indices = np.ctypeslib.as_array((ctypes.c_int32 * max(1, nnz.value)).from_address(ix.value))[: nnz.value].copy()
    lib.gen_free(ip)
    lib.gen_free(ix)
    return indptr, indices


def _dcsbm(cfg: GraphConfig, comm: np.ndarray, sizes: np.ndarray, seed_rng):
    n = cfg.num_nodes
    cbeg = np.zeros(cfg.num_communities + 1, dtype=np.int64)
    np.cumsum(sizes, out=cbeg[1:])
    theta = _power_law(seed_rng, n, 1.0, max(2.0, float(n) ** 0.5), 2.5)
    cum = np.zeros(n + 1, dtype=np.float64)
    np.cumsum(theta, out=cum[1:])
    target = cfg.nnz_target
    scale = target / (2.0 * theta.sum())
    best = None
    for it in range(8):
        indptr, indices = _dcsbm_once(cfg, comm, cbeg, theta, cum, scale, cfg.gen_seed * 131 + it)
        nnz = indices.shape[0]
        err = abs(nnz - target) / target
        if best is None or err < best[0]:
            best = (err, indptr, indices, scale, it)
        if err <= 0.02:
            break
        # duplicates make nnz sub-linear in the stub count: over-correct a little
        ratio = target / max(nnz, 1)
        scale *= ratio ** (1.6 if ratio > 1 else 1.0)
    err, indptr, indices, scale, it = best
    return indptr, indices, {"stub_scale": scale, "iterations": it + 1, "nnz_rel_err": err}


_SM_GAMMA = 0x9E3779B97F4A7C15
_SM_M1 = 0xBF58476D1CE4E5B9
_SM_M2 = 0x94D049BB133111EB


def hash_features(cfg: GraphConfig, rows: np.ndarray) -> np.ndarray:
    """Counter-based features (cfg.device_features): k = splitmix64(key(v, j)) >> 40,
    key = gen_seed * GAMMA + v * F + j (mod 2^64); X[v, j] = k * 2^-23 - 1.  The same formula
    runs on the GPU in ``gen.device.device_features``."""
    rows = np.asarray(rows, dtype=np.uint64)
    f = cfg.feat_dim
    out = np.zeros((rows.shape[0], cfg.feat_ld), dtype=np.float32)
    with np.errstate(over="ignore"):
        base = np.uint64(cfg.gen_seed) * np.uint64(_SM_GAMMA)
        z = base + rows[:, None] * np.uint64(f) + np.arange(f, dtype=np.uint64)[None, :]
        z = z + np.uint64(_SM_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM_M2)
        z = z ^ (z >> np.uint64(31))
    k = (z >> np.uint64(40)).astype(np.float32)
    out[:, :f] = k * np.float32(2.0 ** -23) - np.float32(1.0)
    return out


def make_features(cfg: GraphConfig, rows: Optional[np.ndarray] = None) -> np.ndarray:
    """X[v, j] = k * 2^-23 - 1, k ~ U[0, 2^24) (exact fp32 in [-1, 1)); pad columns zero.

    Generated in row chunks from a chunk-keyed stream so any row range can be
    regenerated independently.  ``rows`` (optional) selects rows."""
    n, f, ld = cfg.num_nodes, cfg.feat_dim, cfg.feat_ld
    if cfg.device_features:
        if rows is None:
            rows = np.arange(n, dtype=np.int64)
        out = np.zeros((len(rows), ld), dtype=np.float32)
        for i in range(0, len(rows), 1 << 18):
            out[i: i + (1 << 18)] = hash_features(cfg, rows[i: i + (1 << 18)])
        return out
    chunk = 1 << 16
    if rows is None:
        out = np.zeros((n, ld), dtype=np.float32)
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            k = _rng(cfg.gen_seed, 1_000_000 + c0 // chunk).integers(0, 1 << 24, size=(c1 - c0, f),
                                                                      dtype=np.int32)
            out[c0:c1, :f] = k.astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
        return out
    rows = np.asarray(rows, dtype=np.int64)
    out = np.zeros((rows.shape[0], ld), dtype=np.float32)
    for ci in np.unique(rows // chunk):
        c0 = int(ci) * chunk
        c1 = min(n, c0 + chunk)
        k = _rng(cfg.gen_seed, 1_000_000 + int(ci)).integers(0, 1 << 24, size=(c1 - c0, f),
                                                            dtype=np.int32)
        sel = np.nonzero(rows // chunk == ci)[0]
        out[sel, :f] = k[rows[sel] - c0].astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
    return out


def _cache_dir(cfg: GraphConfig) -> Optional[str]:
    root = os.environ.get("CMB_GEN_CACHE", "/tmp/cmb_gen_cache")
    if root in ("", "0", "off"):
        return None
    h = hashlib.sha1(repr((GEN_VERSION, asdict(cfg))).encode()).hexdigest()[:16]
    return os.path.join(root, f"{cfg.name.replace('@', '_')}-{h}")


def generate(cfg: GraphConfig, features: bool = True, cache: bool = True) -> Bundle:
    """Deterministic bundle for ``cfg`` (same arrays on every machine/numpy 2.x)."""
    d = _cache_dir(cfg) if (cache and cfg.num_nodes > 100_000) else None
    if d and os.path.exists(os.path.join(d, "done")):
        arr = {k: np.load(os.path.join(d, k + ".npy")) for k in ("indptr", "indices", "comm", "train")}
        meta = dict(np.load(os.path.join(d, "meta.npy"), allow_pickle=True).item())
        b = Bundle(cfg, arr["indptr"], arr["indices"], arr["comm"], arr["train"], None, meta)
    else:
        rng = _rng(cfg.gen_seed, 0)
        sizes = _community_sizes(cfg, rng)
        comm = np.repeat(np.arange(cfg.num_communities, dtype=np.int32), sizes)
        if cfg.kind == "sbm":
            indptr, indices = _sbm(cfg, comm, _rng(cfg.gen_seed, 1))
            meta = {}
        else:
            indptr, indices, meta = _dcsbm(cfg, comm, sizes, _rng(cfg.gen_seed, 1))
        train = np.sort(_rng(cfg.gen_seed, 2).permutation(cfg.num_nodes)[: cfg.n_train]).astype(np.int32)
        src_comm = np.repeat(comm, np.diff(indptr))
        meta.update({
            "num_nodes": cfg.num_nodes, "nnz": int(indices.shape[0]), "nnz_target": cfg.nnz_target,
            "intra_edge_fraction": float(np.mean(src_comm == comm[indices])) if indices.size else 0.0,
            "max_degree": int(np.diff(indptr).max()), "gen_version": GEN_VERSION,
        })
        del src_comm
        b = Bundle(cfg, indptr, indices, comm, train, None, meta)
        if d:  # written under a private name, then renamed: concurrent ranks never see half a cache
            tmp = f"{d}.tmp.{os.getpid()}"
            os.makedirs(tmp, exist_ok=True)
            for k in ("indptr", "indices", "comm", "train"):
                np.save(os.path.join(tmp, k + ".npy"), getattr(b, k))
            np.save(os.path.join(tmp, "meta.npy"), np.array(meta, dtype=object))
            open(os.path.join(tmp, "done"), "w").close()
            try:
                os.rename(tmp, d)
            except OSError:  # another process published it first
                import shutil
                shutil.rmtree(tmp, ignore_errors=True)
    if features and not cfg.device_features:
        b.X = make_features(cfg)
    return b


def feature_rows(bundle: Bundle, rows) -> np.ndarray:
    """X[rows, :F] of the bundle's table (host), also for device-generated tables."""
    cfg = bundle.cfg
    if bundle.X is not None:
        return bundle.X[np.asarray(rows, dtype=np.int64), : cfg.feat_dim]
    return make_features(cfg, np.asarray(rows, dtype=np.int64))[:, : cfg.feat_dim]


def make_labels(bundle: "Bundle", num_classes: int) -> np.ndarray:
    """Synthetic node labels for the training step (NEXT-4): int32 [N] in [0, num_classes),
    homophilous like the paper's datasets -- the community id mod C, replaced by a uniform class
    for 20 % of the nodes (PCG64 stream 7 of the config's seed)."""
    rng = _rng(bundle.cfg.gen_seed, 7)
    n = bundle.comm.shape[0]
    lab = (bundle.comm.astype(np.int64) % num_classes).astype(np.int32)
    flip = rng.random(n) < 0.2
    lab[flip] = rng.integers(0, num_classes, int(flip.sum()), dtype=np.int32)
    return lab
