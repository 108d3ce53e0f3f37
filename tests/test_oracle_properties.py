"""Property-based pins of the oracle (hypothesis, CPU): invariants that must
hold for every input, generated adversarially (many ties, tiny pools, repeated
keys) rather than drawn from the benchmark distribution.  Each property is a
consequence of the definition in SURVEY.md §8(c) / DESIGN.md readings, not a
re-implementation of the oracle:

  S2 top-k (R5/R6): k_eff indices, ascending, -1 padded; every selected
      score >= every unselected one; on equal scores the selected indices are
      the lower ones.
  S3 batch-LRU (R12): every valid selection is resident after the call;
      hits keep their slots; the victims are exactly the k smallest
      (stamp, slot) among the slots not hit with stamp < t; a capacity error
      changes nothing; fwd stays the inverse of slot_key; counts add up.
  S1 score (R2/R3): the fp64 score is an upper bound of every token's
      exact q.k (bound soundness, exact rationals) and lies within the
      sequential-summation error bound of the exact cuboid sum.
"""
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import synth

D = 128
SETTINGS = dict(deadline=None, max_examples=60, suppress_health_check=[HealthCheck.too_slow])


# ----------------------------------------------------------------------------
# S2 top-k
# ----------------------------------------------------------------------------
@settings(**SETTINGS)
@given(st.lists(st.sampled_from([-2.0, -0.0, 0.0, 0.5, 1.0, 1.0, 3.0, 7.5]), min_size=0, max_size=40),
       st.integers(min_value=1, max_value=45))
def test_topk_properties(vals, k):
    n = len(vals)
    max_blk = max(32, ((n + 31) // 32) * 32)
    scores = np.full((1, 1, max_blk), np.nan)
    scores[0, 0, :n] = vals
    sel = oracle.topk(scores, np.array([n], np.int32), k)[0, 0]
    keff = min(k, n)
    chosen = [int(j) for j in sel[:keff]]
    assert (sel[keff:] == -1).all()
    assert chosen == sorted(chosen) and len(set(chosen)) == keff
    assert all(0 <= j < n for j in chosen)
    rest = [j for j in range(n) if j not in set(chosen)]
    if chosen and rest:
        lo = min(vals[j] + 0.0 for j in chosen)
        hi = max(vals[j] + 0.0 for j in rest)
        assert lo >= hi
        if lo == hi:   # ties at the boundary: lower indices win (R5; -0 == +0)
            tied_in = [j for j in chosen if vals[j] + 0.0 == lo]
            tied_out = [j for j in rest if vals[j] + 0.0 == hi]
            assert max(tied_in) < min(tied_out)


# ----------------------------------------------------------------------------
# S3 batch-LRU
# ----------------------------------------------------------------------------
@st.composite
def lru_sequences(draw):
    S = draw(st.integers(min_value=1, max_value=6))
    universe = draw(st.integers(min_value=1, max_value=3 * S + 3))
    calls = []
    for _ in range(draw(st.integers(min_value=1, max_value=12))):
        m = draw(st.integers(min_value=0, max_value=min(universe, S + 2)))
        keys = draw(st.lists(st.integers(min_value=0, max_value=universe - 1), min_size=m, max_size=m, unique=True))
        calls.append(keys)
    return S, universe, calls


@settings(**SETTINGS)
@given(lru_sequences())
def test_batch_lru_properties(case):
    S, universe, calls = case
    fwd_len = universe
    pool = oracle.Pool(S, fwd_len=fwd_len)
    for t, keys in enumerate(calls, start=1):
        before = pool.copy()
        sel = np.array(keys, np.int32).reshape(1, 1, -1) if keys else np.zeros((1, 1, 0), np.int32)
        if sel.shape[2] == 0:
            continue
        r = oracle.lru(pool, sel, np.array([0], np.int32), 0, 1, fwd_len, t)
        hits, misses, evictions, status = r["counts"].tolist()
        hit_keys = [k for k in keys if before.fwd[k] >= 0]
        miss_keys = [k for k in keys if before.fwd[k] < 0]
        hit_slots = {int(before.fwd[k]) for k in hit_keys}
        eligible = sorted((int(before.slot_stamp[s]), s) for s in range(S)
                          if s not in hit_slots and before.slot_stamp[s] < t)
        if len(miss_keys) > len(eligible):
            assert status == 3
            np.testing.assert_array_equal(pool.fwd, before.fwd)
            np.testing.assert_array_equal(pool.slot_key, before.slot_key)
            np.testing.assert_array_equal(pool.slot_stamp, before.slot_stamp)
            continue
        assert status == 0 and hits == len(hit_keys) and misses == len(miss_keys)
        victims = [s for _, s in eligible[:len(miss_keys)]]
        assert evictions == sum(1 for s in victims if before.slot_key[s] != -1)
        out = dict(zip(keys, r["slot"].ravel().tolist()))
        for k in hit_keys:                         # hits keep their slots, re-stamped
            assert out[k] == before.fwd[k] and pool.slot_stamp[out[k]] == t
        assert sorted(out[k] for k in miss_keys) == sorted(victims)   # misses take the LRU victims
        assert [out[k] for k in miss_keys] == victims                 # ... in canonical order
        for k in keys:                               # every selection is resident
            assert pool.fwd[k] == out[k] and pool.slot_key[out[k]] == k
        for s in range(S):                           # untouched slots unchanged
            if s not in hit_slots and s not in victims:
                assert pool.slot_key[s] == before.slot_key[s] and pool.slot_stamp[s] == before.slot_stamp[s]
        for s, key in enumerate(pool.slot_key):      # fwd is the inverse of slot_key
            if key >= 0:
                assert pool.fwd[key] == s
        assert (pool.fwd >= 0).sum() == (pool.slot_key >= 0).sum()


# ----------------------------------------------------------------------------
# S1 score: bound soundness and rounding, exact rationals
# ----------------------------------------------------------------------------
@settings(deadline=None, max_examples=12, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(min_value=0, max_value=2**31 - 1), st.floats(min_value=1e-3, max_value=1e3),
       st.sampled_from([1, 2, 4]))
def test_score_is_sound_upper_bound_within_rounding(seed, scale, G):
    rng = np.random.default_rng(seed)
    nblk = 3
    blocks = synth.encode(synth.kv_blocks(rng, nblk, D) * np.float32(scale), synth.DT_BF16)
    q = synth.encode(rng.standard_normal((1, G, D)), synth.DT_BF16)
    meta = oracle.block_meta(blocks, key_stride=2 * 32 * D).reshape(1, 1, nblk, 2, D)
    s = oracle.block_score(q, meta, np.array([nblk], np.int32))[0, 0]
    qv = [[Fraction(float(x)) for x in synth.decode_f64(q[0, g], synth.DT_BF16)] for g in range(G)]
    for j in range(nblk):
        kv = synth.decode_f64(blocks[j, 0], synth.DT_BF16)          # [32][D]
        mn = synth.decode_f64(meta[0, 0, j, 0], synth.DT_BF16)
        mx = synth.decode_f64(meta[0, 0, j, 1], synth.DT_BF16)
        exact, absum = None, Fraction(0)
        for g in range(G):
            terms = [max(qv[g][c] * Fraction(float(mx[c])), qv[g][c] * Fraction(float(mn[c]))) for c in range(D)]
            tot = sum(terms, Fraction(0))
            exact = tot if exact is None else max(exact, tot)
            absum = max(absum, sum((abs(t) for t in terms), Fraction(0)))
            for tk in range(32):                     # soundness: >= every token's exact q.k
                dot = sum((qv[g][c] * Fraction(float(kv[tk, c])) for c in range(D)), Fraction(0))
                assert Fraction(float(s[j])) >= dot - D * Fraction(2) ** -52 * absum
        # sequential fp64 summation of exact products: |err| <= (D-1) u / (1 - (D-1) u) * sum|t|
        u = Fraction(2) ** -53
        bound = (D - 1) * u / (1 - (D - 1) * u) * absum
        assert abs(Fraction(float(s[j])) - exact) <= bound
