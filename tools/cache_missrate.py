"""NEXT-3 experiment: miss rate of the HBM feature cache (CLOCK, `CAP` rows) in front of the
pinned host table, per Knob setting, over consecutive batches of one epoch (the paper's
S6.5.1 trend: RAND 35.46 % -> MIX-50/25/12.5/0 20.99 / 11.39 / 6.22 / 6.21 % with a
4M-row cache on papers100M).  Prints one JSON object.  Env: CFG (papers100m), CAP (4000000),
BATCHES (300), WARM (50)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402
from gen.device import feature_table  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "papers100m")]
    cap = int(os.environ.get("CAP", "4000000"))
    nbat = int(os.environ.get("BATCHES", "300"))
    warm = int(os.environ.get("WARM", "50"))
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b, features=False)
    t0 = time.time()
    host = torch.empty(cfg.num_nodes, cfg.feat_ld, dtype=torch.float32, pin_memory=True)
    chunk = 1 << 22
    X = feature_table(b, "cuda") if b.X is None else torch.from_numpy(b.X)
    for r0 in range(0, cfg.num_nodes, chunk):
        host[r0: r0 + chunk].copy_(X[r0: r0 + chunk])
    del X
    torch.cuda.synchronize()
    prep_s = time.time() - t0
    out = {"config": cfg.name, "capacity_rows": cap, "batches": nbat, "warmup_batches": warm,
           "host_table_prep_s": round(prep_s, 1), "points": []}
    train = torch.from_numpy(b.train)
    for mode, mix, p in (("rand", 0.0, 0.5), ("comm", 0.5, 1.0), ("comm", 0.25, 1.0),
                         ("comm", 0.125, 1.0), ("comm", 0.0, 1.0), ("norand", 0.0, 1.0)):
        pipe = cmb.MiniBatchPipeline(g, train, cfg.batch_size, cfg.fanouts, mode=mode, mix=mix, p=p)
        s = pipe.sampler
        cache = cmb.FeatureCache(g, host, cfg.feat_dim, max(cap, s.n_cap[-1]), s.n_cap[-1],
                                 s.e_cap[-1])
        pipe.start_epoch(0)
        n = min(nbat, pipe.n_batches)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for t in range(n):
            if t == warm:
                torch.cuda.synchronize()
                cache.stats.zero_()
                e0.record()
            s.sample(pipe.batch_roots(t), p, 42, t)
            s.gather_aggregate_cached(cache)
        e1.record()
        torch.cuda.synchronize()
        rows, miss = cache.stats.tolist()
        ms = e0.elapsed_time(e1)
        out["points"].append({"knob1": mode + (f"(k={mix})" if mode == "comm" else ""),
                              "p_intra": p, "miss_rate": miss / rows,
                              "rows_per_batch": rows / (n - warm),
                              "batches_per_s": (n - warm) / (ms * 1e-3)})
        del cache
    print(json.dumps(out))


if __name__ == "__main__":
    main()
