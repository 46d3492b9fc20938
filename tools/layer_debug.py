"""NEXT-4 bring-up probe: identity weights make Y[:, :F] = bf16(X_dst) and Y[:, F:2F] = bf16(H),
so a wrong descriptor / swizzle / TMEM mapping shows up as a recognisable permutation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2504_18082_b200 as cmb
from gen import CONFIGS, generate, scaled

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
cfg = CONFIGS[name] if name == "tiny" else scaled(CONFIGS[name], 0.01)
b = generate(cfg); F = cfg.feat_dim; fo = 256
g = cmb.Graph.from_bundle(b)
ws = torch.zeros(F, fo); wn = torch.zeros(F, fo)
for c in range(F):
    ws[c, c] = 1.0
    if F + c < fo: wn[c, F + c] = 1.0
layer = cmb.SageLayer(ws, wn, None, relu=False)
order = oracle.order_roots(b.train, b.comm, cfg.num_communities, 0, 0.0, 42, 0)
roots = oracle.batch_roots(order, cfg.batch_size, 0)
s = cmb.Sampler(g, len(roots), cfg.fanouts)
view = s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, 42, 0)
y = s.sage_layer(layer); torch.cuda.synchronize()
print("status", s.status())
n, e = view.host_sizes(); L = len(cfg.fanouts); nd = n[L - 1]
x_in, h = s.gather_aggregate(); torch.cuda.synchronize()
xd = x_in[:nd, :F].to(torch.bfloat16).float().cpu().numpy()
hh = h[:nd, :F].to(torch.bfloat16).float().cpu().numpy()
yg = y[:nd].cpu().numpy()
print("nd", nd, "self ok", np.array_equal(yg[:, :F], xd), "neigh ok",
      np.array_equal(yg[:, F:F + min(F, fo - F)], hh[:, :min(F, fo - F)]))
np.set_printoptions(linewidth=200, precision=3, suppress=True)
print("y[0,:24]", yg[0, :24]); print("x[0,:24]", xd[0, :24])
print("y[9,:24]", yg[9, :24]); print("x[9,:24]", xd[9, :24])
# locate where each of y's first-row values comes from
for r in (0, 1, 8, 33):
    for c in (0, 1, 5, 8, 9):
        v = yg[r, c]
        hits = np.argwhere(xd == v)[:3] if v != 0 else []
        print(f"y[{r},{c}]={v:.4f} found in xd at {hits.tolist() if len(hits) else '-'}")
