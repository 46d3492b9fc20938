"""Effective L2 capacity probe for random 400-B feature rows (B200).

Mean-of-5 aggregation (cmb_sage_mean_aggregate) whose 5*nd source ids are drawn uniformly from
a random subset of S rows of the products-shaped table: every row of the subset is touched
~868K/S times, so once the subset fits in L2 the reads stop costing DRAM.  Prints
{S_MB: us per launch, GB/s of row reads} -- the knee is the L2 capacity this access stream
actually gets."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402
from microbench_gather import timeit  # noqa: E402


def main():
    cfg = CONFIGS["products"]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    X = g.features
    F = cfg.feat_dim
    R = 4 * F
    N = cfg.num_nodes
    refs = 868_000
    nd = refs // 5
    ip = torch.arange(0, 5 * nd + 1, 5, dtype=torch.int32, device="cuda")
    ndv = torch.tensor([nd], dtype=torch.int64, device="cuda")
    acc = torch.empty(nd, g.feat_ld, device="cuda")
    out = {}
    # per-row vs per-byte cost with L2-resident rows (8-MB scattered subset): row width sweep
    S = 8_000_000 // R
    subset = torch.randperm(N, device="cuda")[:S]
    ids = subset[torch.randint(0, S, (5 * nd,), device="cuda")].to(torch.int32)
    for f in (16, 32, 64, 100):
        ms = timeit(lambda: cmb.sage_mean_aggregate(ip, ids, ndv, X, f, acc))
        out[f"l2res_ld100_f{f}"] = {"us": round(ms * 1e3, 1),
                                    "read_GBs": round(5 * nd * 4 * f / ms / 1e6, 1)}
    X128 = torch.randn(N // 8, 128, device="cuda")
    ids2 = torch.randint(0, 8_000_000 // 512, (5 * nd,), device="cuda").to(torch.int32)
    acc2 = torch.empty(nd, 128, device="cuda")
    for f in (32, 64, 96, 128):
        ms = timeit(lambda: cmb.sage_mean_aggregate(ip, ids2, ndv, X128, f, acc2))
        out[f"l2res_ld128_f{f}"] = {"us": round(ms * 1e3, 1),
                                    "read_GBs": round(5 * nd * 4 * f / ms / 1e6, 1)}
    # access ORDER with L2-resident rows: sequential ids (i mod S) vs random ids
    seq = (torch.arange(5 * nd, device="cuda") % S).to(torch.int32)
    ms = timeit(lambda: cmb.sage_mean_aggregate(ip, seq, ndv, X, F, acc))
    out["l2res_sequential_f100"] = {"us": round(ms * 1e3, 1),
                                    "read_GBs": round(5 * nd * R / ms / 1e6, 1)}
    # plain streaming reads from L2 (torch reduction over a 32-MB tensor)
    t = torch.randn(8_000_000, device="cuda")
    ms = timeit(lambda: t.sum())
    out["l2res_torch_sum_32MB"] = {"us": round(ms * 1e3, 1), "read_GBs": round(32e6 / ms / 1e6, 1)}
    t2 = torch.randn(100_000_000, device="cuda")
    ms = timeit(lambda: t2.sum())
    out["dram_torch_sum_400MB"] = {"us": round(ms * 1e3, 1), "read_GBs": round(400e6 / ms / 1e6, 1)}
    print(json.dumps(out))
    return
    for kind in ("scattered", "contiguous"):
        for mb in (8, 32, 64, 96, 128, 192, 256, 384, 512, 980):
            S = min(N, mb * 1_000_000 // R)
            if kind == "scattered":   # S rows spread over the whole table (all its 2-MB pages)
                subset = torch.randperm(N, device="cuda")[:S]
            else:                     # the first S rows (S*R bytes of pages)
                subset = torch.arange(S, device="cuda")
            ids = subset[torch.randint(0, S, (5 * nd,), device="cuda")].to(torch.int32)
            ms = timeit(lambda: cmb.sage_mean_aggregate(ip, ids, ndv, X, F, acc))
            out[f"{kind}_{mb}"] = {"us": round(ms * 1e3, 1),
                                   "read_GBs": round(5 * nd * R / ms / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
