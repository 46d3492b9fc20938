"""Row-gather bandwidth probes on the products-shaped feature table (B200).

Times (CUDA events, median of reps) several ways of moving U rows of X:
  cmb gather (random ids), cmb gather (sorted ids), torch index_select (random ids),
  contiguous copy of U rows (streaming), cmb fused gather+aggregate of a real batch.
Prints one JSON object.  Used to find the attainable bandwidth for random 400-B rows.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def timeit(fn, reps=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    X = g.features
    F = cfg.feat_dim
    R = 4 * F
    N = cfg.num_nodes
    out = {}
    for U in (200_000, 576_000, 1_000_000):
        ids = torch.randperm(N, device="cuda")[:U].to(torch.int32)
        sids = torch.sort(ids).values
        n_dev = torch.tensor([U], dtype=torch.int64, device="cuda")
        o = torch.empty(U, g.feat_ld, device="cuda")
        r = {}
        ms = timeit(lambda: cmb.gather_features(g, ids, n_dev, o))
        r["cmb_gather_random"] = 2 * U * R / ms / 1e6
        ms = timeit(lambda: cmb.gather_features(g, sids, n_dev, o))
        r["cmb_gather_sorted"] = 2 * U * R / ms / 1e6
        idl = ids.long()
        ms = timeit(lambda: torch.index_select(X, 0, idl, out=o))
        r["torch_index_select_random"] = 2 * U * R / ms / 1e6
        src = X[:U]
        ms = timeit(lambda: o.copy_(src))
        r["contiguous_copy"] = 2 * U * g.feat_ld * 4 / ms / 1e6
        # mostly-read: mean of 5 random rows per dst (reads U rows, writes U/5 rows)
        nd = U // 5
        acc = torch.empty(nd, g.feat_ld, device="cuda")
        ip = torch.arange(0, 5 * nd + 1, 5, dtype=torch.int32, device="cuda")
        ndv = torch.tensor([nd], dtype=torch.int64, device="cuda")
        ms = timeit(lambda: cmb.sage_mean_aggregate(ip, ids, ndv, X, F, acc))
        r["cmb_mean5_random"] = (5 * nd + nd) * R / ms / 1e6
        out[f"U={U}"] = {k: round(v, 1) for k, v in r.items()}
    out["unit"] = "GB/s (algorithmic bytes: rows read + rows written)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
