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


def device_features(cfg, device, chunk_rows: int = 1 << 20, row_begin: int = 0,
                    row_end: int = None) -> torch.Tensor:
    """Rows [row_begin, row_end) of the table (default: all of it) -- a row shard is generated
    in place on its own GPU."""
    n, f, ld = cfg.num_nodes, cfg.feat_dim, cfg.feat_ld
    row_end = n if row_end is None else min(n, int(row_end))
    row_begin = min(int(row_begin), row_end)
    X = torch.zeros(max(1, row_end - row_begin), ld, dtype=torch.float32, device=device)
    base = (cfg.gen_seed * _SM_GAMMA) % (1 << 64)
    cols = torch.arange(f, dtype=torch.int64, device=device)
    for r0 in range(row_begin, row_end, chunk_rows):
        r1 = min(row_end, r0 + chunk_rows)
        v = torch.arange(r0, r1, dtype=torch.int64, device=device)
        z = v[:, None] * f + cols[None, :]
        z = z + _i64((base + _SM_GAMMA) % (1 << 64))
        z = (z ^ _shr(z, 30)) * _i64(_SM_M1)
        z = (z ^ _shr(z, 27)) * _i64(_SM_M2)
        z = z ^ _shr(z, 31)
        k = _shr(z, 40).to(torch.float32)
        X[r0 - row_begin:r1 - row_begin, :f] = k * (2.0 ** -23) - 1.0
    return X


def feature_table(bundle: Bundle, device, row_begin: int = 0, row_end: int = None) -> torch.Tensor:
    """The bundle's feature table on `device`, or its rows [row_begin, row_end) (a shard)."""
    n = bundle.cfg.num_nodes
    row_end = n if row_end is None else min(n, int(row_end))
    if bundle.X is not None:
        if row_begin == 0 and row_end == n:
            return torch.from_numpy(bundle.X).to(device)
        return torch.from_numpy(bundle.X[row_begin:max(row_end, row_begin + 1)]).to(device)
    return device_features(bundle.cfg, device, row_begin=row_begin, row_end=row_end)
