"""NEXT-1 on one GPU: fused gather+aggregate time, replicated table vs W virtual shards read
through the pointer table (products-shaped, RAND p = 0.5).  Prints one JSON object."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    X = g.features
    pipe = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts, p=0.5)
    pipe.start_epoch(0)
    s = pipe.sampler
    out = {}
    for W in (1, 2, 4, 8):
        S = (cfg.num_nodes + W - 1) // W
        shards = [X[r * S: (r + 1) * S].clone() for r in range(W)]
        table = cmb.ShardTable(shards, cfg.num_nodes, cfg.feat_dim)
        ts_d, ts_s = [], []
        for t in range(30):
            s.sample(pipe.batch_roots(t), 0.5, 42, t)
            for which, ts in (("dense", ts_d), ("sharded", ts_s)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if which == "dense":
                    s.gather_aggregate()
                else:
                    s.gather_aggregate_sharded(table)
                e1.record()
                torch.cuda.synchronize()
                if t >= 5:
                    ts.append(e0.elapsed_time(e1) * 1e3)
        out[f"W={W}"] = {"dense_us": round(float(np.median(ts_d)), 1),
                         "sharded_us": round(float(np.median(ts_s)), 1)}
        del shards, table
    print(json.dumps(out))


if __name__ == "__main__":
    main()
