"""Feature tables on the GPU (input generation, not the method).

``device_features`` produces the same bytes as ``planted.hash_features`` (splitmix64 of a
counter, numpy uint64 there, torch int64 with masked logical shifts here) directly in HBM,
so a papers100M-sized table (57 GB) never exists on the host.  ``feature_table`` returns
the device table of any bundle."""
from __future__ import annotations

import torch

from .planted import _SM_GAMMA, _SM_M1, _SM_M2, Bundle


def _i64(u: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    return u - (1 << 64) if u >= 1 << 63 else u


def _shr(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def device_features(cfg, device, chunk_rows: int = 1 << 20) -> torch.Tensor:
    n, f, ld = cfg.num_nodes, cfg.feat_dim, cfg.feat_ld
    X = torch.zeros(n, ld, dtype=torch.float32, device=device)
    base = (cfg.gen_seed * _SM_GAMMA) % (1 << 64)
    cols = torch.arange(f, dtype=torch.int64, device=device)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        v = torch.arange(r0, r1, dtype=torch.int64, device=device)
        z = v[:, None] * f + cols[None, :]
        z = z + _i64((base + _SM_GAMMA) % (1 << 64))
        z = (z ^ _shr(z, 30)) * _i64(_SM_M1)
        z = (z ^ _shr(z, 27)) * _i64(_SM_M2)
        z = z ^ _shr(z, 31)
        k = _shr(z, 40).to(torch.float32)
        X[r0:r1, :f] = k * (2.0 ** -23) - 1.0
    return X


def feature_table(bundle: Bundle, device) -> torch.Tensor:
    if bundle.X is not None:
        return torch.from_numpy(bundle.X).to(device)
    return device_features(bundle.cfg, device)
