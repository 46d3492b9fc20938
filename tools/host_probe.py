"""Host-side enqueue cost of one BatchedPipeline group (4 batches) vs the GPU time of the group,
products MIX-0 / p = 1 (short kernels) and RAND / p = 0.5."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def main():
    cfg = CONFIGS["products"]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    out = {}
    for mode, mix, p in (("comm", 0.0, 1.0), ("rand", 0.0, 0.5)):
        pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                                   mode=mode, mix=mix, p=p, nb=4)
        pipe.step_group(range(4))
        torch.cuda.synchronize()
        for ev in (False, True):
            G = 40
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record()
            for k in range(G):
                pipe.step_group(range(4 * k, 4 * k + 4), events={} if ev else None)
            t1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            out[f"{mode}{mix}_p{p}_events{int(ev)}"] = {
                "host_us_per_group": round((t1 - t0) / G * 1e6, 1),
                "gpu_us_per_group": round(e0.elapsed_time(e1) / G * 1e3, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
