"""The knob effect on the dominant kernel, per (Knob-1, Knob-2) point (north_star: "ncu counters
(achieved HBM GB/s against the B200 peak, L2 hit rate and unique-feature bytes per batch,
reported against Knob-1/Knob-2)"; the paper's per-epoch effect).

Plain run: per knob point, BATCHES consecutive batches of epoch 0 through MiniBatchPipeline;
prints one JSON line per point with device-timed sample and gather+aggregate ms, unique input
rows and bytes per batch.  Under `ncu --metrics ... -k regex:k_gather_mean_row` the same
launches are captured in order (BATCHES per point, after WARM warm-up batches per point), and
tools/knob_counters_summary.py joins the two.  Env: CFG (products), BATCHES (8), WARM (2)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402
from gen.device import feature_table  # noqa: E402

POINTS = {
    # BASELINE configs[1]: "Knob-1 uniform vs community"
    "arxiv": [("rand", 0.0, 0.9), ("comm", 0.5, 0.9), ("comm", 0.125, 0.9), ("comm", 0.0, 0.9),
              ("norand", 0.0, 0.9)],
    # configs[2]: "p_intra sweep 0.5-1.0" (RAND roots and community roots)
    "reddit": [("rand", 0.0, p) for p in (0.5, 0.6, 0.7, 0.8, 0.9, 1.0)] +
              [("comm", 0.0, p) for p in (0.5, 0.75, 1.0)],
    # configs[3]: the paper's per-epoch comparison points
    "products": [("rand", 0.0, 0.5), ("comm", 0.5, 0.5), ("comm", 0.0, 0.5), ("norand", 0.0, 0.5),
                 ("comm", 0.125, 1.0), ("comm", 0.0, 1.0), ("norand", 0.0, 1.0)],
}


def main():
    name = os.environ.get("CFG", "products")
    nbat = int(os.environ.get("BATCHES", "8"))
    warm = int(os.environ.get("WARM", "2"))
    cfg = CONFIGS[name]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b, features=feature_table(b, "cuda"))
    L = len(cfg.fanouts)
    F = cfg.feat_dim
    s = torch.cuda.current_stream()
    for mode, mix, p in POINTS[name]:
        pipe = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                                     mode=mode, mix=mix, p=p, seed=42)
        pipe.start_epoch(0)
        smp = pipe.sampler
        for k in range(warm):
            smp.sample(pipe.batch_roots(k), p, 42, k)
            smp.gather_aggregate()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(nbat)]
        sizes = torch.zeros(nbat, 2 * L + 1, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        for k in range(nbat):
            bi = warm + k
            ev[k][0].record(s)
            smp.sample(pipe.batch_roots(bi), p, 42, bi)
            ev[k][1].record(s)
            smp.gather_aggregate()
            ev[k][2].record(s)
            sizes[k].copy_(smp.sizes, non_blocking=True)
        torch.cuda.synchronize()
        sz = sizes.cpu().numpy()
        U, nd, ed = sz[:, L], sz[:, L - 1], sz[:, L + 1 + L - 1]
        R = 4 * F
        alg = 2 * U * R + nd * R + 4 * ed + 4 * (nd + 1) + 4 * U
        print(json.dumps({
            "config": name, "knob1": mode + (f"(k={mix})" if mode == "comm" else ""),
            "p_intra": p, "batches": nbat, "warm": warm,
            "sample_ms": float(np.mean([e[0].elapsed_time(e[1]) for e in ev])),
            "gather_aggregate_ms": float(np.mean([e[1].elapsed_time(e[2]) for e in ev])),
            "unique_input_rows": float(U.mean()), "unique_feature_bytes": float(U.mean() * R),
            "edges_last_hop": float(ed.mean()), "algorithmic_bytes": float(alg.mean())}),
            flush=True)


if __name__ == "__main__":
    main()
