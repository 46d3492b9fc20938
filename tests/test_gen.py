"""The seeded input generators (gen/): the host and device feature formulas agree bit for bit,
and the table has the documented value set (exact fp32 k * 2^-23 - 1, k < 2^24)."""
import numpy as np
import torch

from gen import CONFIGS, scaled
from gen.device import device_features
from gen.planted import hash_features, make_features


def test_device_features_match_host_formula():
    cfg = scaled(CONFIGS["papers100m"], 0.0002)
    Xd = device_features(cfg, "cpu", chunk_rows=4096).numpy()
    Xh = hash_features(cfg, np.arange(cfg.num_nodes))
    assert Xd.tobytes() == Xh.tobytes()
    rows = np.array([0, 7, cfg.num_nodes - 1, 12345 % cfg.num_nodes])
    assert make_features(cfg, rows).tobytes() == Xh[rows].tobytes()


def test_hash_feature_values():
    cfg = scaled(CONFIGS["papers100m"], 0.0002)
    X = hash_features(cfg, np.arange(2000))
    F = cfg.feat_dim
    k = (X[:, :F].astype(np.float64) + 1.0) * 2.0 ** 23
    assert np.all(k == np.round(k)) and k.min() >= 0 and k.max() < 2 ** 24
    assert np.all(X[:, F:] == 0)
    assert abs(float(X[:, :F].mean())) < 0.01        # ~U[-1, 1)
    assert abs(float(X[:, :F].std()) - 1 / np.sqrt(3)) < 0.01
    assert torch.from_numpy(X).isfinite().all()


def test_device_feature_shards_concatenate_to_the_table():
    # bench.py --shard: rank r generates rows [r*S, (r+1)*S) in place; the shards are the table
    from types import SimpleNamespace
    from gen.device import feature_table
    cfg = scaled(CONFIGS["papers100m"], 0.0002)
    full = device_features(cfg, "cpu", chunk_rows=1000).numpy()
    W = 3
    S = (cfg.num_nodes + W - 1) // W
    parts = [device_features(cfg, "cpu", chunk_rows=1000, row_begin=r * S,
                             row_end=(r + 1) * S).numpy() for r in range(W)]
    assert np.concatenate(parts).tobytes() == full.tobytes()
    host = SimpleNamespace(cfg=scaled(CONFIGS["products"], 0.001), X=None)
    host.X = make_features(host.cfg)
    sh = feature_table(host, "cpu", 10, 25).numpy()
    assert sh.tobytes() == host.X[10:25].tobytes()
