"""batches/s of the products workload: sequential pipeline vs the overlapped one (sampler of
batch k+1 concurrent with gather+aggregate of batch k).  Env knobs of libcmb apply."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def timed(fn, K):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    fn(K)
    b.record(s)
    torch.cuda.synchronize()
    return K / (a.elapsed_time(b) * 1e-3)


def main():
    cfg = CONFIGS["products"]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    K = int(os.environ.get("K", "200"))
    seq = cmb.MiniBatchPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts, p=0.5)
    ov = cmb.OverlappedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts, p=0.5,
                                depth=int(os.environ.get("DEPTH", "2")))

    def run_seq(K):
        for t in range(K):
            seq.step(t)

    def run_ov(K):
        for t in range(K):
            ov.step(t)
        ov.join()

    bats = {nb: cmb.BatchedPipeline(g, torch.from_numpy(b.train), cfg.batch_size, cfg.fanouts,
                                    p=0.5, nb=nb) for nb in (2, 4)}

    def run_bat(nb):
        def f(K):
            for t in range(0, K, nb):
                bats[nb].step_group(range(t, t + nb))
        return f

    run_seq(10)
    run_ov(10)
    for nb in bats:
        run_bat(nb)(8)
    out = {"seq": timed(run_seq, K), "overlap": timed(run_ov, K)}
    for nb in bats:
        out[f"batched{nb}"] = timed(run_bat(nb), K)
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
