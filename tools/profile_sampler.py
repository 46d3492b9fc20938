"""Sub-step timeline of the persistent sampler kernel.

Every block's thread 0 writes %globaltimer at fixed sub-step boundaries into the workspace
(sample_persist.cuh CMB_PROF).  For each sub-step this prints the critical-path increment
dT = max_b t_b[k] - max_b t_b[k-1] and the mean / max per-block duration (microseconds),
averaged over a few batches of the chosen workload (env CFG, P, MODE, MIX)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402

PROF_OFFSET = 115200         # carve order: header 256, barrier 256, pub 3*4096*8, dst-order
                             # hist 4096*4 (sample.cu)
SUB = ["relabel(h-1)", "count", "prefix", "positions", "picks+mark", "barrierA",
       "flag_scan", "prefix2", "assign", "barrierC"]


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    p = float(os.environ.get("P", cfg.p_intra))
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    nb = int(os.environ.get("NB", "1"))  # batches per sampler launch (BatchedPipeline)
    pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                               mode=os.environ.get("MODE", "rand"),
                               mix=float(os.environ.get("MIX", "0")), p=p, nb=nb)
    L = len(cfg.fanouts)
    # 32-bit map words: the last hop relabels inside its assign step (no final barrier) and has
    # one more stamp after the dst-order placement
    npts = 2 + 10 * L
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nblk = (sms - sms % nb) // nb  # virtual blocks of batch 0 of each launch
    labels = [f"h{h}.{s}" for h in range(L - 1) for s in SUB]
    for x in SUB[:-1]:
        if x == "flag_scan":
            labels.append(f"h{L - 1}.place_dst_rows")
        labels.append(f"h{L - 1}.{x}")
    labels.append("end")
    crit, mean, mx = [], [], []
    pipe.start_epoch(0)
    for t in range(25):
        pipe.step_group(list(range(t * nb, t * nb + nb)))
        torch.cuda.synchronize()
        ws = pipe.sampler.workspace
        raw = ws[PROF_OFFSET: PROF_OFFSET + nblk * 64 * 8].view(torch.int64).cpu().numpy()
        tb = raw.reshape(nblk, 64)[:, :npts].astype(np.float64)
        if t >= 5:
            T = tb.max(axis=0)
            crit.append(np.diff(T) / 1e3)
            d = np.diff(tb, axis=1) / 1e3
            mean.append(d.mean(axis=0))
            mx.append(d.max(axis=0))
    crit, mean, mx = (np.mean(x, axis=0) for x in (crit, mean, mx))
    rows = {lab: [round(float(c), 2), round(float(m), 2), round(float(x), 2)]
            for lab, c, m, x in zip(labels, crit, mean, mx)}
    print(json.dumps({"unit": "us [critical dT, mean block, max block]", "total_us":
                      round(float(crit.sum()), 1), "steps": rows,
                      "sizes": pipe.sampler.sizes.cpu().tolist()}))


if __name__ == "__main__":
    main()
