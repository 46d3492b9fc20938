"""Where the step's time goes between kernels: the bench's launch-group loop (products, RAND,
p = 0.5, cmb.DEFAULT_BATCHES_PER_LAUNCH batches per group) with CUDA events around the sampler
launch, the gather launch and the per-group sizes copy, and the gap from one group's last event
to the next group's first (microseconds per group, averaged)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402
from gen.device import feature_table  # noqa: E402


def main():
    G = int(os.environ.get("NB", cmb.DEFAULT_BATCHES_PER_LAUNCH))
    cfg = CONFIGS["products"]
    b = generate(cfg)
    dev = torch.device("cuda:0")
    g = cmb.Graph.from_bundle(b, device=dev, features=feature_table(b, dev))
    pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts, p=0.5,
                               nb=G)
    L = len(cfg.fanouts)
    nbat = pipe.n_batches
    K = 396 // G * G
    for t in range(0, 8 * G, G):
        pipe.step_group([t + i for i in range(G)])
    torch.cuda.synchronize()
    sizes_log = torch.zeros(K, 2 * L + 1, dtype=torch.int64, device=dev)
    evs = [pipe.make_events(G) for _ in range(0, K, G)]
    cp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(0, K, G)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for q, k0 in enumerate(range(0, K, G)):
        pipe.step_group([(8 * G + k0 + i) % nbat for i in range(G)], events=evs[q])
        cp[q][0].record()
        sizes_log[k0:k0 + G].copy_(pipe.group_sizes[:G], non_blocking=True)
        cp[q][1].record()
    t1.record()
    torch.cuda.synchronize()
    ng = len(evs)
    samp = sum(e[0].elapsed_time(e[1]) for e in evs) / ng * 1e3
    gath = sum(e[2].elapsed_time(e[-1]) for e in evs) / ng * 1e3
    s2g = sum(e[1].elapsed_time(e[2]) for e in evs) / ng * 1e3
    copy = sum(c[0].elapsed_time(c[1]) for c in cp) / ng * 1e3
    g2c = sum(e[-1].elapsed_time(c[0]) for e, c in zip(evs, cp)) / ng * 1e3
    c2n = sum(cp[q][1].elapsed_time(evs[q + 1][0]) for q in range(ng - 1)) / (ng - 1) * 1e3
    print(json.dumps({"batches_per_group": G, "us_per_group": t0.elapsed_time(t1) / ng * 1e3,
                      "sampler": samp, "sampler_to_gather": s2g, "gather": gath,
                      "gather_to_copy": g2c, "sizes_copy": copy, "copy_to_next_group": c2n}))


if __name__ == "__main__":
    main()
