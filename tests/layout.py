"""Test-side helpers: storage conversions and the tiled-metadata permutation
(include/sparseserve.h "Metadata layout").  Pure reshapes/transposes; no
method arithmetic."""
import numpy as np
import torch

import synth

D = 128


def to_torch(a: np.ndarray, device="cuda") -> torch.Tensor:
    """numpy storage (uint16 bf16 bits / float32 / ints) -> torch tensor."""
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def to_numpy(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def cpc(storage_dtype) -> int:
    return 8 if np.dtype(storage_dtype) == np.uint16 else 4


def tiled_to_logical(tiled: np.ndarray, B: int, Hkv: int, max_blk: int) -> np.ndarray:
    """tiled flat array -> logical [B][Hkv][max_blk][2][d]."""
    c = cpc(tiled.dtype)
    nchk = D // c
    t = tiled.reshape(B, Hkv, max_blk // 32, nchk, 2, 32, c)
    t = t.transpose(0, 1, 2, 5, 4, 3, 6)            # [B][Hkv][tiles][r][mm][chunk][e]
    return np.ascontiguousarray(t).reshape(B, Hkv, max_blk, 2, D)


def logical_to_tiled(logical: np.ndarray) -> np.ndarray:
    B, Hkv, max_blk, _, _ = logical.shape
    c = cpc(logical.dtype)
    nchk = D // c
    t = logical.reshape(B, Hkv, max_blk // 32, 32, 2, nchk, c)
    t = t.transpose(0, 1, 2, 5, 4, 3, 6)            # [B][Hkv][tiles][chunk][mm][r][e]
    return np.ascontiguousarray(t).reshape(-1)


def storage(dtype_name: str):
    return np.uint16 if dtype_name == synth.DT_BF16 else np.float32


def mean_tiled_to_logical(tiled: np.ndarray, B: int, Hkv: int, max_blk: int) -> np.ndarray:
    """NEXT-3 float32 mean metadata: tiled [..][tiles][d/4][32][4] -> [B][Hkv][max_blk][d]."""
    t = tiled.reshape(B, Hkv, max_blk // 32, D // 4, 32, 4).transpose(0, 1, 2, 4, 3, 5)
    return np.ascontiguousarray(t).reshape(B, Hkv, max_blk, D)


def mean_logical_to_tiled(logical: np.ndarray) -> np.ndarray:
    B, Hkv, max_blk, _ = logical.shape
    t = logical.reshape(B, Hkv, max_blk // 32, 32, D // 4, 4).transpose(0, 1, 2, 4, 3, 5)
    return np.ascontiguousarray(t).reshape(-1)
