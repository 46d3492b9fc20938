"""The five synthetic workload shapes (BASELINE.json ``configs``).

Node/edge/feature counts follow the paper's Table 2 and
OGB's ogbn-arxiv; fanouts are in HOP order (index 0 = the hop that expands the
roots; reading R6).  ``nnz_target`` counts CSR entries of the
symmetrised graph (reading R16: Table 2 "#Edges" = CSR entries).
"""
from dataclasses import dataclass, replace
from typing import Tuple


@dataclass(frozen=True)
class GraphConfig:
    name: str
    num_nodes: int
    nnz_target: int
    num_communities: int
    comm_size_range: Tuple[int, int]
    mu: float                 # fraction of stubs that leave their community
    feat_dim: int
    feat_ld: int              # row stride in floats; ld*4 is a multiple of 16 B
    n_train: int
    batch_size: int
    fanouts: Tuple[int, ...]  # hop order
    p_intra: float            # default Knob-2 value of the config
    gen_seed: int
    kind: str = "dcsbm"       # "sbm" (plain stochastic block model) or "dcsbm"
    # features from a counter-based hash, generated on the GPU (the 57-GB papers100M table is
    # never materialised on the host); rows for the oracle come from the same formula in numpy
    device_features: bool = False


_S = 250418082  # gen_seed base; + config index

CONFIGS = {
    # configs[0]: plain SBM, 8 x 125 nodes, p_in = 9/124, p_out = 1/875 -> mean degree 10
    "tiny": GraphConfig("tiny", 1_000, 10_000, 8, (125, 125), 0.1, 16, 16, 600, 64,
                        (5, 5), 0.9, _S + 0, kind="sbm"),
    # configs[1]: ogbn-arxiv shape (169,343 nodes, 1,166,243 undirected edges)
    "arxiv": GraphConfig("arxiv", 169_343, 2_332_486, 256, (64, 8_192), 0.25, 128, 128,
                         90_941, 1024, (15, 10, 5), 0.9, _S + 1),
    # configs[2]: reddit shape (Table 2 row 1)
    "reddit": GraphConfig("reddit", 232_965, 114_615_892, 256, (128, 16_384), 0.3, 602, 604,
                          153_431, 1024, (25, 10), 0.9, _S + 2),
    # configs[3]: ogbn-products shape (Table 2 row 3)
    "products": GraphConfig("products", 2_449_029, 123_718_280, 2_048, (128, 65_536), 0.2, 100,
                            100, 196_615, 1024, (15, 10, 5), 0.5, _S + 3),
    # configs[4]: ogbn-papers100M shape (Table 2 row 4)
    "papers100m": GraphConfig("papers100m", 111_059_956, 3_228_124_712, 65_536, (256, 262_144),
                              0.2, 128, 128, 1_207_179, 1024, (15, 10, 5), 0.5, _S + 4,
                              device_features=True),
}


def scaled(cfg: GraphConfig, factor: float, name: str = None) -> GraphConfig:
    """Same shape (mean degree, mu, F, fanouts, train fraction), ``factor`` x the nodes.

    Used for parity tests that must finish in seconds on the oracle while still
    spanning many tiles and a ragged tail."""
    n = max(64, int(cfg.num_nodes * factor))
    deg = cfg.nnz_target / cfg.num_nodes
    c = max(2, int(cfg.num_communities * factor ** 0.5))
    lo, hi = cfg.comm_size_range
    lo = max(4, min(lo, n // (2 * c)))
    hi = max(lo + 1, min(hi, n // 2))
    ntr = max(1, int(cfg.n_train * factor))
    return replace(cfg, name=name or f"{cfg.name}@{factor:g}", num_nodes=n,
                   nnz_target=int(n * min(deg, 0.5 * (n - 1))), num_communities=c,
                   comm_size_range=(lo, hi), n_train=ntr)


# class counts of the paper's datasets (Table 2: ogbn-arxiv 40, reddit 41,
# ogbn-products 47, ogbn-papers100M 172); tiny is a test size
NUM_CLASSES = {"tiny": 8, "arxiv": 40, "reddit": 41, "products": 47, "papers100m": 172}


def num_classes(cfg: GraphConfig) -> int:
    return NUM_CLASSES.get(cfg.name.split("@")[0].split("_")[0], 8)
