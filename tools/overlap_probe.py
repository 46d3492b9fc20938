"""batches/s of the products workload (RAND, p = 0.5): the bench's sequential launch groups
(4 batches per sampler launch, then their 4 fused gathers, one stream) versus double-buffered
groups on two streams (the sampler of group k+1 concurrent with the gathers of group k).
Prints one JSON line; run under different libcmb env knobs to A/B the resource split."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb  # noqa: E402
from gen import CONFIGS, generate  # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "products")]
    b = generate(cfg)
    g = cmb.Graph.from_bundle(b)
    K = int(os.environ.get("K", "400"))
    p = float(os.environ.get("P", "0.5"))
    train = torch.from_numpy(b.train)
    bat = cmb.BatchedPipeline(g, train, cfg.batch_size, cfg.fanouts, p=p, nb=4)
    bat.start_epoch(0)
    sets = [[bat.samplers[i] for i in range(4)],
            [cmb.Sampler(g, cfg.batch_size, cfg.fanouts) for _ in range(4)]]
    for ss in sets:
        for s in ss:
            s.alloc_features()
    s_s, s_g = torch.cuda.Stream(), torch.cuda.Stream()
    ev_s = [torch.cuda.Event() for _ in range(2)]
    ev_g = [torch.cuda.Event() for _ in range(2)]
    nb = bat.n_batches

    def roots(t):
        return [bat.batch_roots((t + i) % nb) for i in range(4)]

    def seq(n):
        for t in range(0, n, 4):
            bat.step_group([(t + i) % nb for i in range(4)])

    def ovl(n):
        cur = torch.cuda.current_stream()
        s_s.wait_stream(cur)
        s_g.wait_stream(cur)
        for q, t in enumerate(range(0, n, 4)):
            j = q & 1
            with torch.cuda.stream(s_s):
                s_s.wait_event(ev_g[j])
                cmb.sample_multi(sets[j], roots(t), [(t + i) % nb for i in range(4)], p, 42)
                ev_s[j].record(s_s)
            with torch.cuda.stream(s_g):
                s_g.wait_event(ev_s[j])
                for s in sets[j]:
                    s.gather_aggregate()
                ev_g[j].record(s_g)
        cur.wait_stream(s_s)
        cur.wait_stream(s_g)

    def only_sample(n):
        for t in range(0, n, 4):
            cmb.sample_multi(sets[0], roots(t), [(t + i) % nb for i in range(4)], p, 42)

    def only_gather(n):
        for t in range(0, n, 4):
            for s in sets[0]:
                s.gather_aggregate()

    def timed(fn):
        fn(16)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(K)
        e.record()
        torch.cuda.synchronize()
        return a.elapsed_time(e) * 1e3 / K  # us per batch

    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("CMB_")},
           "seq_us": timed(seq), "overlap_us": timed(ovl),
           "sample_only_us": timed(only_sample), "gather_only_us": timed(only_gather)}
    for k in ("seq_us", "overlap_us"):
        out[k.replace("_us", "_bps")] = 1e6 / out[k]
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
