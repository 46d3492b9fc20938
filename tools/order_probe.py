"""Does the visiting order of the last hop's dst rows change the fused gather's time / DRAM
traffic?  products-shaped input: per batch (sampled with the dst order on), the fused a4 + a5
kernel in the natural order, in the sampler's bucketed order (cmb_blocks.dst_order) and through
the one-shard ShardedRows map.  Checks the bytes are identical, prints the mean kernel time per
form (CUDA events).  Under ncu, -k regex:k_gather_mean_row gives the DRAM bytes of each launch
(launch order per batch: natural, sampler_order, sharded1)."""
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
    b = generate(cfg)
    from gen.device import feature_table
    g = cmb.Graph.from_bundle(b, features=feature_table(b, "cuda"))
    L = len(cfg.fanouts)
    out = {}
    for mode, mix, p in ((os.environ.get("MODE", "rand"), float(os.environ.get("MIX", "0")),
                          float(os.environ.get("P", "0.5"))),):
        pipe = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                                     mode=mode, mix=mix, p=p)
        pipe.start_epoch(0)
        s = pipe.sampler
        t = {k: [] for k in ("natural", "sampler_order", "sharded1")}
        table = cmb.ShardTable([g.features], cfg.num_nodes, cfg.feat_dim)
        same = True
        for k in range(K):
            s.set_dst_order(True)
            s.sample(pipe.batch_roots(k), p, 42, k)
            n = int(s.sizes[L - 1].item())
            ref = None
            for name in t:
                s.set_dst_order(name == "sampler_order")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                x_in, h = (s.gather_aggregate_sharded(table) if name == "sharded1" else
                           s.gather_aggregate())
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
            s.set_dst_order(True)
        out[f"{mode}({mix})|{p}"] = {k: sum(v) / len(v) for k, v in t.items()}
        out[f"{mode}({mix})|{p}"]["bytes_identical"] = same
    print(json.dumps(out))


if __name__ == "__main__":
    main()
