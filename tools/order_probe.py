"""Does the visiting order of the last hop's dst rows change the fused gather's DRAM traffic?
products-shaped input: per batch, the fused a4 + a5 kernel in the natural order and with
dst_order = (a) rows sorted by node id, (b) sorted by id >> SHIFT buckets (stable), (c) a random
permutation (control).  Checks the bytes are identical to the natural order's, prints the mean
kernel time per order (CUDA events).  Under ncu, -k regex:k_gather_mean_row gives the DRAM
bytes of each launch (launch order: natural, sorted, bucketed, random per batch)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    K = int(os.environ.get("K", "24"))
    shift = int(os.environ.get("SHIFT", "10"))
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    L = len(cfg.fanouts)
    out = {}
    for mode, mix, p in ((os.environ.get("MODE", "rand"), float(os.environ.get("MIX", "0")),
                          float(os.environ.get("P", "0.5"))),):
        pipe = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                                     mode=mode, mix=mix, p=p)
        pipe.start_epoch(0)
        s = pipe.sampler
        t = {k: [] for k in ("natural", "sorted", "bucketed", "random", "sharded1")}
        table = cmb.ShardTable([g.features], cfg.num_nodes, cfg.feat_dim)
        same = True
        gen = torch.Generator(device="cuda").manual_seed(0)
        for k in range(K):
            s.sample(pipe.batch_roots(k), p, 42, k)
            n = int(s.sizes[L - 1].item())
            nodes = s.nodes[:n]
            orders = {"natural": None,
                      "sorted": torch.argsort(nodes, stable=True).to(torch.int32),
                      "bucketed": torch.argsort(nodes >> shift, stable=True).to(torch.int32),
                      "random": torch.randperm(n, device="cuda", generator=gen).to(torch.int32),
                      "sharded1": "sharded1"}
            ref = None
            for name, o in orders.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                x_in, h = (s.gather_aggregate_sharded(table) if isinstance(o, str) else
                           s.gather_aggregate(o))
                e1.record()
                torch.cuda.synchronize()
                if k >= 2:
                    t[name].append(e0.elapsed_time(e1) * 1e3)
                nl = int(s.sizes[L].item())
                cur = (x_in[:nl].clone(), h[:n].clone())
                if ref is None:
                    ref = cur
                else:
                    same &= bool(torch.equal(ref[0], cur[0]) and torch.equal(ref[1], cur[1]))
        out[f"{mode}({mix})|{p}"] = {k: sum(v) / len(v) for k, v in t.items()}
        out[f"{mode}({mix})|{p}"]["bytes_identical"] = same
    print(json.dumps(out))


if __name__ == "__main__":
    main()
