"""NEXT-1 (second half) experiment: fraction of a batch's input rows that live in ANOTHER rank's
feature shard (a6 row sharding, S = ceil(N / W)), under round-robin batch -> rank placement
(b mod W, reading R22) versus the community-aware shard-aligned placement
(dist.aligned_schedule), per Knob setting.  Remote rows are what the one-sided sharded gather
reads over NVLink (or what the a6 all-to-all moves).  Counts only -- one GPU samples every batch
and the owner arithmetic is exact.  Prints one JSON object.  Env: CFG (papers100m), WORLD (8),
BATCHES (64 evenly spaced batches of epoch 0)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402
from paper_2504_18082_b200 import dist as cmb_dist  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "papers100m")]
    world = int(os.environ.get("WORLD", "8"))
    nbat = int(os.environ.get("BATCHES", "64"))
    t0 = time.time()
    b = generate(cfg, features=False)
    g = cmb.Graph.from_bundle(b, features=False)
    S = (cfg.num_nodes + world - 1) // world
    out = {"config": cfg.name, "world": world, "rows_per_shard": S, "batches_sampled": nbat,
           "gen_s": round(time.time() - t0, 1), "points": []}
    train = torch.from_numpy(b.train)
    L = len(cfg.fanouts)
    for mode, mix, p in (("rand", 0.0, 0.5), ("comm", 0.5, 1.0), ("comm", 0.125, 1.0),
                         ("comm", 0.0, 1.0), ("norand", 0.0, 1.0)):
        pipe = cmb.MiniBatchPipeline(g, train, cfg.batch_size, cfg.fanouts, mode=mode, mix=mix, p=p)
        pipe.start_epoch(0)
        nb = pipe.n_batches
        sched = cmb_dist.aligned_schedule(pipe.order, cfg.batch_size, cfg.num_nodes, world)
        rank_of = {bb: r for r, bs in enumerate(sched) for bb in bs}
        rr, al, home_hits = [], [], 0
        for bi in np.linspace(0, nb - 1, min(nbat, nb)).astype(int):
            view = pipe.sampler.sample(pipe.batch_roots(int(bi)), p, 42, int(bi))
            n, _ = view.host_sizes()
            U = n[L]
            rr.append(cmb_dist.remote_fraction(view.nodes, U, int(bi) % world, S))
            al.append(cmb_dist.remote_fraction(view.nodes, U, rank_of[int(bi)], S))
            roots = pipe.batch_roots(int(bi)).cpu().numpy()
            home_hits += int(int(np.median(roots)) // S == rank_of[int(bi)])
        out["points"].append({
            "knob1": mode + (f"(k={mix})" if mode == "comm" else ""), "p_intra": p,
            "remote_fraction_round_robin": float(np.mean(rr)),
            "remote_fraction_aligned": float(np.mean(al)),
            "batches_on_home_rank": home_hits / len(al),
            "per_rank_batches": [len(x) for x in sched]})
        print(json.dumps(out["points"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
