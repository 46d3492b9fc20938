"""batches/s of the products step (RAND, p = 0.5) at nb batches per sampler launch, for a library
built with a larger CMB_MAX_BATCHES_PER_LAUNCH (layout experiment; env NB, CMB_LIB_PATH)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def main():
    nb = int(os.environ.get("NB", "4"))
    cmb.MAX_BATCHES_PER_LAUNCH = max(cmb.MAX_BATCHES_PER_LAUNCH, nb)
    cfg = CONFIGS["products"]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    mode = os.environ.get("MODE", "rand")  # Knob-1 (env MODE, MIX, P)
    pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                               mode=mode, mix=float(os.environ.get("MIX", "0")),
                               p=float(os.environ.get("P", "0.5")), nb=nb)
    K = 400 // nb * nb
    for t in range(0, 8 * nb, nb):
        pipe.step_group(list(range(t, t + nb)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [pipe.make_events(nb) for _ in range(0, K, nb)]
    e0.record()
    for q, t in enumerate(range(0, K, nb)):
        pipe.step_group([(t + i) % pipe.n_batches for i in range(nb)], events=ev[q])
    e1.record()
    torch.cuda.synchronize()
    samp = sum(e[0].elapsed_time(e[1]) for e in ev) / K * 1e3
    gath = sum(e[1].elapsed_time(e[-1]) for e in ev) / K * 1e3
    print(json.dumps({"nb": nb, "us_per_batch": e0.elapsed_time(e1) / K * 1e3,
                      "sample_us": samp, "gather_us": gath}))


if __name__ == "__main__":
    main()
