"""Training-step probe (products): per-step device time of sample + train_step over K batches;
under ncu the launch list shows each kernel's share."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate, make_labels, num_classes, scaled  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    if os.environ.get("SCALE"):
        cfg = scaled(cfg, float(os.environ["SCALE"]))
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    C = num_classes(cfg)
    labels = torch.from_numpy(make_labels(b, C)).cuda()
    pipe = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts, p=0.5)
    pipe.start_epoch(0)
    smp = pipe.sampler
    model = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=len(cfg.fanouts), seed=1)
    K = int(os.environ.get("K", "20"))
    for k in range(min(3, pipe.n_batches)):
        smp.sample(pipe.batch_roots(k), 0.5, 42, k)
        model.train_step(smp, labels)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        smp.sample(pipe.batch_roots(k % pipe.n_batches), 0.5, 42, k)
        model.train_step(smp, labels)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e3 * (t1 - t0) / K:.3f} ms/step, wall {1e3 * (t2 - t0) / K:.3f} ms/step")


if __name__ == "__main__":
    main()
