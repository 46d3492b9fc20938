import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18082_b200 as cmb
import oracle
from gen import CONFIGS, generate, scaled
cfg = scaled(CONFIGS["products"], 0.01)
b = generate(cfg)
g = cmb.Graph.from_bundle(b)
F, L, fo = cfg.feat_dim, len(cfg.fanouts), 256
gen = torch.Generator().manual_seed(5)
layer = cmb.SageLayer(torch.randn(F, fo, generator=gen) / 10, torch.randn(F, fo, generator=gen) / 10,
                      torch.zeros(fo), relu=True, out_bf16=True)
order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, 42, 0)
roots = oracle.batch_roots(order, cfg.batch_size, 1)
s = cmb.Sampler(g, len(roots), cfg.fanouts)
s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, 42, 1)
y = s.sage_layer(layer, save_a=True)
dy = torch.randn(s.n_cap[L - 1], fo, device="cuda") * 0.01
r = []
for saved in (False, False, True, True):
    r.append([t.clone() for t in s.sage_layer_backward(layer, dy, y, saved=saved)])
torch.cuda.synchronize()
for i, j in ((0, 1), (2, 3), (0, 2)):
    for k in range(3):
        d = (r[i][k] - r[j][k]).abs()
        print(i, j, k, float(d.max()), int((d > 0).sum()), tuple(torch.nonzero(d > 0)[:3].tolist()))
nd = int(s.sizes[L - 1].item())
print("n_dst", nd, "tiles", (nd + 127) // 128)
for i in range(4):
    for k in range(3):
        assert torch.equal(r[0][k].view(torch.int32), r[i][k].view(torch.int32)), (i, k)
print("all four bit-identical")
