"""NEXT-4 backward bring-up probe: per-(half, feature block) error of dW against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2504_18082_b200 as cmb
from gen import CONFIGS, generate, scaled
name = sys.argv[1]
fo = int(sys.argv[2])
cfg = CONFIGS[name] if name == "tiny" else scaled(CONFIGS[name], 0.01)
b = generate(cfg); prep = oracle.graph_prep(b); g = cmb.Graph.from_bundle(b)
F = cfg.feat_dim
layer = cmb.SageLayer(torch.zeros(F, fo), torch.zeros(F, fo), None, relu=False, out_bf16=True)
order = oracle.order_roots(b.train, b.comm, cfg.num_communities, 0, 0.0, 42, 0)
roots = oracle.batch_roots(order, cfg.batch_size, 1)
s = cmb.Sampler(g, len(roots), cfg.fanouts)
s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, 42, 1)
ref = oracle.run_batch(prep, b.X, F, roots, cfg.fanouts, cfg.p_intra, 42, 1)
L = len(cfg.fanouts); nd = ref["n"][L - 1]
Xd = ref["X_in"][:nd, :F].astype(np.float64); H = ref["H64"][:, :F]
dY = torch.ones(s.n_cap[L - 1], fo, dtype=torch.bfloat16, device="cuda")
dY[nd:] = 0
dws, dwn, db = s.sage_layer_backward(layer, dY)
torch.cuda.synchronize()
rs, rn, rb = oracle.sage_conv_backward(Xd, H, np.ones((nd, fo)))
print("nd", nd, "tiles", (nd + 127) // 128, "grid env", os.environ.get("CMB_BWD_GRID"))
for nm, got, r in (("self", dws, rs), ("neigh", dwn, rn)):
    got = got.double().cpu().numpy()
    e = np.abs(got - r) / (np.abs(r) + 1e-3)
    for f0 in range(0, F, 16):
        print(nm, f0, "max rel err %.3g" % e[f0:f0 + 16].max(), "col0 got %.4f ref %.4f" % (got[f0, 0], r[f0, 0]))
print("db", db[:4].cpu().numpy(), rb[:4])
