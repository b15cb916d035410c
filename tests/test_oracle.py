"""Pins for the float64 oracle (oracle/decode_attention_ref.c) — CPU only.

Each test checks the oracle against something other than itself: closed forms,
invariants that the mathematics fixes, an arbitrary-precision brute force
(mpmath, 50 digits), a library routine (torch SDPA in float64), the numpy
fp16/bf16 decoders, and a hand-derived golden example (tests/golden/).
Chosen so that a dropped term, wrong sign/index or transposed operand fails.
"""
import json
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import synth
from oracle import attention as oa

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, rng, amp=1.0):
    # values on the generator's 24-bit lattice (exact in fp32 and float64)
    return (rng.integers(-(1 << 23), 1 << 23, size=shape) * 2.0 ** -22 * amp).astype(np.float64)


def _run(q, ks, vs, dtype="f64", scale=None):
    return oa.decode_attention(q, ks, vs, dtype, scale=scale, nthreads=2)


# ---------------------------------------------------------------- decoders

def test_f16_decoder_all_bit_patterns():
    bits = np.arange(1 << 16, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oa.decode_element(int(b), "f16") for b in bits])
    finite = np.isfinite(ref)
    assert np.array_equal(got[finite], ref[finite])
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(got[np.isinf(ref)], ref[np.isinf(ref)])


def test_bf16_decoder_all_bit_patterns():
    bits = np.arange(1 << 16, dtype=np.uint16)
    ref = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    got = np.array([oa.decode_element(int(b), "bf16") for b in bits])
    finite = np.isfinite(ref)
    assert np.array_equal(got[finite], ref[finite])
    assert np.array_equal(np.isnan(got), np.isnan(ref))


# ---------------------------------------------------------------- closed forms

def test_ctx1_returns_v0_exactly():
    rng = np.random.default_rng(1)
    q = _rand((1, 4, 16), rng)
    k = _rand((1, 2, 16), rng)
    v = _rand((1, 2, 16), rng)
    out = _run(q, [k], [v])
    for h in range(4):
        assert np.array_equal(out[0, h], v[0, h // 2])


def test_identical_keys_give_mean_of_v():
    rng = np.random.default_rng(2)
    n, D = 37, 32
    k = np.repeat(_rand((1, 1, D), rng), n, axis=0)
    v = _rand((n, 1, D), rng)
    q = _rand((1, 1, D), rng, amp=8)
    out = _run(q, [k], [v])
    np.testing.assert_allclose(out[0, 0], v[:, 0].mean(axis=0), rtol=0, atol=1e-13)


def test_zero_query_gives_mean_of_v():
    rng = np.random.default_rng(3)
    k = _rand((50, 2, 16), rng)
    v = _rand((50, 2, 16), rng)
    out = _run(np.zeros((1, 2, 16)), [k], [v])
    for h in range(2):
        np.testing.assert_allclose(out[0, h], v[:, h].mean(axis=0), rtol=0, atol=1e-13)


def test_constant_v_rows_return_that_row():
    rng = np.random.default_rng(4)
    c = _rand((1, 1, 24), rng)
    v = np.repeat(c, 33, axis=0)
    out = _run(_rand((1, 1, 24), rng, 8), [_rand((33, 1, 24), rng)], [v])
    np.testing.assert_allclose(out[0, 0], c[0, 0], rtol=1e-14, atol=1e-15)


def test_softmax_weights_sum_to_one():
    for dtype in ("f32", "f16", "bf16"):
        q = synth.gen_rows(0, 0, [0], [0], 4, 128, dtype, amp=8)
        k = synth.gen_seq(1, 0, 0, 777, 2, 128, dtype)
        for h in range(4):
            w = oa.attention_weights(q[0, h], k, h // 2, dtype)
            assert abs(w.sum() - 1.0) < 1e-12
            assert (w >= 0).all()


def test_dominant_token_selects_its_value():
    # key j aligned with q, all others orthogonal -> score gap >= 40 -> out = v_j + O(n e^-40)
    D, n, j = 16, 20, 7
    q = np.zeros((1, 1, D)); q[0, 0, 3] = 40.0 * math.sqrt(D)
    k = np.zeros((n, 1, D)); k[j, 0, 3] = 1.0
    rng = np.random.default_rng(5)
    v = _rand((n, 1, D), rng)
    out = _run(q, [k], [v])
    np.testing.assert_allclose(out[0, 0], v[j, 0], rtol=0, atol=n * math.exp(-40) * 2 + 1e-15)


def test_two_token_logistic_closed_form():
    # n=2: w0 = 1/(1+exp(s1-s0)) (logistic), out = w0 v0 + (1-w0) v1
    rng = np.random.default_rng(6)
    D = 8
    q = _rand((1, 1, D), rng, 4); k = _rand((2, 1, D), rng); v = _rand((2, 1, D), rng)
    s = [float(np.dot(q[0, 0], k[t, 0])) / math.sqrt(D) for t in range(2)]
    w0 = 1.0 / (1.0 + math.exp(s[1] - s[0]))
    expect = w0 * v[0, 0] + (1 - w0) * v[1, 0]
    np.testing.assert_allclose(_run(q, [k], [v])[0, 0], expect, rtol=1e-13, atol=1e-15)


def test_golden_hand_derived_example():
    with open(os.path.join(GOLDEN, "attention_hand_derived.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        q = np.array(c["q"], dtype=np.float64)[None]
        k = np.array(c["K"], dtype=np.float64)
        v = np.array(c["V"], dtype=np.float64)
        out = _run(q, [k], [v], scale=c.get("scale"))
        np.testing.assert_allclose(out[0], np.array(c["out"]), rtol=0, atol=c["atol"])


# ---------------------------------------------------------------- invariants

def test_token_permutation_invariance():
    rng = np.random.default_rng(7)
    k = _rand((64, 2, 32), rng); v = _rand((64, 2, 32), rng); q = _rand((1, 4, 32), rng, 8)
    perm = rng.permutation(64)
    a = _run(q, [k], [v]); b = _run(q, [k[perm]], [v[perm]])
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-14)


def test_linearity_in_v():
    rng = np.random.default_rng(8)
    k = _rand((40, 1, 16), rng); v = _rand((40, 1, 16), rng); q = _rand((1, 1, 16), rng, 8)
    alpha, c = -1.75, _rand((1, 1, 16), rng)
    a = _run(q, [k], [alpha * v + c])
    b = alpha * _run(q, [k], [v]) + c[0]
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)


def test_gqa_equals_mha_with_repeated_kv():
    rng = np.random.default_rng(9)
    Hq, Hkv, D, n = 8, 2, 16, 45
    q = _rand((1, Hq, D), rng, 8); k = _rand((n, Hkv, D), rng); v = _rand((n, Hkv, D), rng)
    gqa = _run(q, [k], [v])
    rep = Hq // Hkv
    mha = _run(q, [np.repeat(k, rep, axis=1)], [np.repeat(v, rep, axis=1)])
    assert np.array_equal(gqa, mha)        # same arithmetic, same order -> identical


def test_gqa_mapping_is_consecutive_groups():
    # q-head h must read kv head h // (Hq/Hkv): perturbing kv head 1 changes heads 2,3 only
    rng = np.random.default_rng(10)
    q = _rand((1, 4, 8), rng, 8); k = _rand((9, 2, 8), rng); v = _rand((9, 2, 8), rng)
    a = _run(q, [k], [v])
    v2 = v.copy(); v2[:, 1] += 1.0
    b = _run(q, [k], [v2])
    assert np.array_equal(a[0, :2], b[0, :2])
    np.testing.assert_allclose(b[0, 2:], a[0, 2:] + 1.0, rtol=0, atol=1e-13)


def test_ragged_batch_rows_independent_and_row_subset():
    rng = np.random.default_rng(11)
    ns = [1, 17, 300]
    ks = [_rand((n, 2, 16), rng) for n in ns]; vs = [_rand((n, 2, 16), rng) for n in ns]
    q = _rand((3, 4, 16), rng, 8)
    full = _run(q, ks, vs)
    for b in range(3):
        single = _run(q[b:b + 1], [ks[b]], [vs[b]])
        assert np.array_equal(full[b], single[0])
    rows = np.array([11, 0, 5])
    sub = oa.decode_attention(q, ks, vs, "f64", rows=rows, nthreads=3)
    for i, r in enumerate(rows):
        assert np.array_equal(sub[i], full[r // 4, r % 4])


def test_rejects_empty_context():
    with pytest.raises(ValueError):
        _run(np.zeros((1, 1, 4)), [np.zeros((0, 1, 4))], [np.zeros((0, 1, 4))])


# ---------------------------------------------------------------- brute force / library

@settings(max_examples=40, deadline=None)
@given(n=st.integers(1, 8), D=st.integers(1, 8), hkv=st.sampled_from([1, 2]),
       g=st.sampled_from([1, 2]), amp=st.sampled_from([1.0, 8.0]), seed=st.integers(0, 2**31))
def test_vs_mpmath_tiny(n, D, hkv, g, amp, seed):
    import mpmath
    mpmath.mp.dps = 50
    rng = np.random.default_rng(seed)
    Hq = hkv * g
    q = _rand((1, Hq, D), rng, amp); k = _rand((n, hkv, D), rng); v = _rand((n, hkv, D), rng)
    out = _run(q, [k], [v])
    scale = 1 / mpmath.sqrt(D)
    for h in range(Hq):
        kv = h // g
        s = [scale * mpmath.fsum(mpmath.mpf(q[0, h, d]) * mpmath.mpf(k[t, kv, d]) for d in range(D))
             for t in range(n)]
        e = [mpmath.exp(x) for x in s]
        z = mpmath.fsum(e)
        for d in range(D):
            ref = mpmath.fsum(e[t] * mpmath.mpf(v[t, kv, d]) for t in range(n)) / z
            assert abs(out[0, h, d] - float(ref)) <= 1e-12 * (1 + abs(float(ref)))


@pytest.mark.parametrize("Hq,Hkv,n,dtype", [(32, 32, 512, "f32"), (8, 2, 333, "bf16"),
                                            (4, 4, 100, "f16"), (32, 8, 1000, "bf16")])
def test_vs_torch_sdpa_float64(Hq, Hkv, n, dtype):
    import torch
    D = 128
    q = synth.gen_rows(0, 0, [0], [n - 1], Hq, D, dtype, amp=8)
    k = synth.gen_seq(1, 0, 0, n, Hkv, D, dtype)
    v = synth.gen_seq(2, 0, 0, n, Hkv, D, dtype)
    out = oa.decode_attention(q, [k], [v], dtype, nthreads=4)

    def widen(a):  # independent widening via numpy's float16 / bit views
        if dtype == "f32":
            return a.astype(np.float64)
        if dtype == "f16":
            return a.view(np.float16).astype(np.float64)
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

    tq = torch.from_numpy(widen(q)).permute(1, 0, 2).unsqueeze(0)             # [1,Hq,1,D]
    tk = torch.from_numpy(widen(k)).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0).unsqueeze(0)
    tv = torch.from_numpy(widen(v)).permute(1, 0, 2).repeat_interleave(Hq // Hkv, 0).unsqueeze(0)
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)[0, :, 0].numpy()
    np.testing.assert_allclose(out[0], ref, rtol=1e-12, atol=1e-13)
