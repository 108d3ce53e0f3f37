"""NEXT-2 parity: the incremental working-set tracker (union
of the blocks selected over the past w = 12 decoding steps) against the oracle's
or_ws_estimate (the union written from its definition, pinned in
tests/test_oracle_pins.py) on the same selections, over many steps, several
layers and heads."""
import numpy as np
import pytest
import torch

import oracle
from layout import to_torch

pytestmark = pytest.mark.gpu


def test_ws_track_equals_set_union():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200 import ops
    rng = np.random.default_rng(11)
    L, B, Hkv, k, max_blk, w = 3, 4, 2, 16, 200, 12
    st = ops.WorkingSetState(L, B, Hkv, max_blk, k, w)
    d = ops.dims(B, Hkv, Hkv)
    steps = []                         # [t] -> [L][B][Hkv][k] selections
    prev = {}
    for t in range(40):
        step = np.full((L, B, Hkv, k), -1, np.int32)
        for l in range(L):
            sel = np.full((B, Hkv, k), -1, np.int32)
            for b in range(B):
                for h in range(Hkv):
                    kk = int(rng.integers(1, k + 1))
                    old = prev.get((l, b, h), [])
                    keep = set(rng.choice(old, size=min(len(old), kk // 2), replace=False).tolist()) if old else set()
                    while len(keep) < kk:
                        keep.add(int(rng.integers(0, max_blk)))
                    s = sorted(keep)[:kk]
                    sel[b, h, :len(s)] = s
                    prev[(l, b, h)] = s
            step[l] = sel
            ops.ws_track(st, l, to_torch(sel), k, d, max_blk, t)
        steps.append(step)
        torch.cuda.synchronize()
        got = st.ws_count.cpu().numpy()
        exp = oracle.ws_estimate(np.stack(steps), max_blk, w)[t]
        assert (got == exp).all(), (t, got, exp)
