"""Pins of the oracle's RoPE (the paper's Query/KeyTransform, "fuse normalization, RoPE",
P:329-338 StreamingLLM fused RoPE; R31: rotate-half pairs (i, i + D/2),
theta_i = rope_theta^(-2i/D) / rope_scale, key t at position t, query row r at l_kv - l_qo + r).

What fixes it independently of the C code: the rotation at position 0 is the identity; it
preserves each pair's norm; in 2-D it is the textbook rotation by pos*theta; scores depend only
on the position difference (Su et al.'s defining property) — checked on single vectors and at
attention level, where prepending masked keys shifts every position; and the C oracle equals a
NumPy brute force written as complex multiplication. A negative control shows the interleaved
pairing convention would be caught. CPU only."""
import numpy as np
import pytest

import oracle
import synth

THETA = 10000.0


def test_rotation_identity_at_position_zero():
    x = np.random.default_rng(0).normal(size=128)
    assert np.array_equal(oracle.rope_rotate(x, 0, THETA), x)


@pytest.mark.parametrize("pos", [1, 17, 4095, 524287])
def test_rotation_preserves_pair_norms(pos):
    x = np.random.default_rng(pos).normal(size=128)
    y = oracle.rope_rotate(x, pos, THETA)
    n0 = x[:64] ** 2 + x[64:] ** 2
    n1 = y[:64] ** 2 + y[64:] ** 2
    assert np.max(np.abs(n0 - n1)) < 1e-12


def test_two_dim_textbook_rotation_and_scale():
    # D = 2: theta_0 = 1 / rope_scale; (1, 0) -> (cos a, sin a), (0, 1) -> (-sin a, cos a)
    for pos, sc in ((3, 1.0), (100, 4.0)):
        a = pos / sc
        assert np.allclose(oracle.rope_rotate([1.0, 0.0], pos, THETA, sc), [np.cos(a), np.sin(a)], atol=1e-15)
        assert np.allclose(oracle.rope_rotate([0.0, 1.0], pos, THETA, sc), [-np.sin(a), np.cos(a)], atol=1e-15)
    # frequency of pair i is theta^(-2i/D): pair 1 of D = 4 turns by pos * theta^(-1/2)
    y = oracle.rope_rotate([0.0, 1.0, 0.0, 0.0], 7, THETA)
    a = 7 * THETA ** -0.5
    assert np.allclose(y, [0.0, np.cos(a), 0.0, np.sin(a)], atol=1e-15)
    # position interpolation: (pos, scale s) == (pos / s, scale 1)
    x = np.random.default_rng(1).normal(size=64)
    assert np.max(np.abs(oracle.rope_rotate(x, 800, THETA, 8.0) - oracle.rope_rotate(x, 100, THETA, 1.0))) < 1e-12


@pytest.mark.parametrize("shift", [1, 64, 100000])
def test_scores_depend_only_on_position_difference(shift):
    r = np.random.default_rng(shift)
    q, k = r.normal(size=128), r.normal(size=128)
    for p, t in ((5, 0), (4000, 3999), (17, 30)):
        a = oracle.rope_rotate(q, p, THETA) @ oracle.rope_rotate(k, t, THETA)
        b = oracle.rope_rotate(q, p + shift, THETA) @ oracle.rope_rotate(k, t + shift, THETA)
        assert abs(a - b) < 1e-9 * max(1.0, abs(a))


def _rope(wl, theta=THETA, scale=1.0):
    import dataclasses
    return dataclasses.replace(wl, rope_theta=theta, rope_scale=scale)


@pytest.mark.parametrize("seed", range(12))
def test_c_oracle_equals_complex_brute_force(seed):
    r = np.random.default_rng(700 + seed)
    B = int(r.integers(1, 4))
    H_kv = int(r.choice([1, 2]))
    g = int(r.choice([1, 4]))
    D = int(r.choice([32, 64, 128]))
    ps = int(r.choice([1, 4, 16]))
    mask = ["none", "causal"][seed % 2]
    kv = r.integers(1, 70, B).astype(np.int32)
    qo = np.minimum(r.integers(1, 5, B), kv).astype(np.int32)
    wl = _rope(synth.Workload("rope", H_kv * g, H_kv, D, ps, "bf16", mask, qo, kv), scale=[1.0, 2.0][seed % 2])
    inp = synth.make_inputs(wl, seed_base=seed)
    a = oracle.attention_from_inputs(inp)
    b = oracle.brute_force_from_inputs(inp)
    assert np.max(np.abs(a[0] - b[0])) < 1e-12 and np.max(np.abs(a[1] - b[1])) < 1e-12
    # RoPE changes the result (the transform is really applied)
    c = oracle.attention_from_inputs(synth.make_inputs(_rope(wl, 0.0), seed_base=seed))
    if int(kv.max()) > 1:
        assert np.max(np.abs(a[1] - c[1])) > 1e-3


def _raw(n_keys, q, K, V, mask_bits=None):
    """One request, page size 1, the C oracle with RoPE (1 head, D from q)."""
    D = q.size
    lk = n_keys
    kw = dict(mask="none")
    if mask_bits is not None:
        kw = dict(mask="custom", custom_mask=np.packbits(mask_bits.astype(np.uint8), bitorder="little"),
                  mask_bit_indptr=np.array([0, lk], np.int64))
    return oracle.paged_attention(
        qo_indptr=np.array([0, 1], np.int32), kv_page_indptr=np.array([0, lk], np.int32),
        kv_last_page_len=np.array([1], np.int32), kv_page_indices=np.arange(lk, dtype=np.int32),
        q=q.astype(np.float32).reshape(1, 1, D), k_pool=K.astype(np.float32).reshape(lk, 1, 1, D),
        v_pool=V.astype(np.float32).reshape(lk, 1, 1, D), k_strides=(D, D, D), v_strides=(D, D, D), H_qo=1, H_kv=1,
        D=D, page_size=1, dtype="f32", sm_scale=0.125, rope_theta=THETA, **kw)


@pytest.mark.parametrize("s", [1, 5, 300])
def test_attention_invariant_to_prepended_masked_keys(s):
    """Prepending s keys and masking them out shifts every key position AND the query position
    (right-aligned, R4/R31) by s: the output must not change. Pins the position conventions."""
    r = np.random.default_rng(s)
    n, D = 9, 64
    q, K, V = r.normal(size=D), r.normal(size=(n, D)), r.uniform(-1, 1, size=(n, D))
    a = _raw(n, q, K, V)
    K2 = np.concatenate([r.normal(size=(s, D)), K])
    V2 = np.concatenate([r.uniform(-1, 1, size=(s, D)), V])
    bits = np.concatenate([np.zeros(s, bool), np.ones(n, bool)])
    b = _raw(n + s, q, K2, V2, bits)
    # equal up to the f32 rounding of the transformed q / k (R31); a wrong position convention
    # moves o and lse by O(0.1)
    assert np.max(np.abs(a[0] - b[0])) < 1e-5 and abs(a[1][0, 0] - b[1][0, 0]) < 1e-5


def test_single_key_at_position_zero_is_unrotated():
    # position 0 rotates by 0: q, k pass through exactly (f32 inputs round to themselves)
    r = np.random.default_rng(3)
    q, K, V = r.normal(size=32), r.normal(size=(1, 32)), r.uniform(-1, 1, size=(1, 32))
    o, lse = _raw(1, q, K, V)
    assert np.array_equal(o[0, 0], V[0].astype(np.float32).astype(np.float64))
    assert abs(lse[0, 0] - 0.125 * float(q.astype(np.float32).astype(np.float64) @ K[0].astype(np.float32))) < 1e-12


def test_interleaved_pairing_would_be_caught():
    """Negative control: the GPT-J pairing (2i, 2i+1) gives different attention, so the pins above
    distinguish the two conventions."""
    wl = _rope(synth.Workload("rope", 4, 1, 64, 4, "bf16", "none", np.array([1], np.int32), np.array([40], np.int32)))
    inp = synth.make_inputs(wl)
    ref = oracle.attention_from_inputs(inp)
    from synth import raw_bits
    q = oracle.to_float64(raw_bits(inp.q), "bf16").reshape(-1, 4, 64)
    perm = np.concatenate([np.arange(0, 64, 2), np.arange(1, 64, 2)])  # interleaved -> rotate-half order
    inv = np.argsort(perm)
    bf = oracle.brute_force(
        qo_indptr=inp.qo_indptr, kv_page_indptr=inp.kv_page_indptr, kv_last_page_len=inp.kv_last_page_len,
        kv_page_indices=inp.kv_page_indices.numpy(), q=raw_bits(inp.q), k_pool=raw_bits(inp.k_pool),
        v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=4, H_kv=1, D=64,
        page_size=4, dtype="bf16", sm_scale=inp.sm_scale, rope_theta=THETA)
    assert np.max(np.abs(bf[1] - ref[1])) < 1e-12
    # the same data with the pairs laid out interleaved: permuting d before a rotate-half RoPE and
    # back is what an interleaved implementation computes
    del q, inv
    qp = raw_bits(inp.q).reshape(-1, 4, 64)[..., perm].copy()
    kp = raw_bits(inp.k_pool).reshape(-1, 4, 1, 64)[..., perm].copy()
    inter = oracle.brute_force(
        qo_indptr=inp.qo_indptr, kv_page_indptr=inp.kv_page_indptr, kv_last_page_len=inp.kv_last_page_len,
        kv_page_indices=inp.kv_page_indices.numpy(), q=qp, k_pool=kp, v_pool=raw_bits(inp.v_pool),
        k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=4, H_kv=1, D=64, page_size=4, dtype="bf16",
        sm_scale=inp.sm_scale, rope_theta=THETA)
    assert np.max(np.abs(inter[1] - ref[1])) > 1e-3


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
def test_transform_output_rounding(dtype):
    """R31: the transformed q / k are tensors of the input dtype (round to nearest, ties to even).
    The C oracle's rounding against numpy's own float types / an f64-bit-pattern bf16 rounding,
    and against torch's bf16 conversion."""
    import torch
    r = np.random.default_rng(5)
    x = r.normal(size=3000) * np.exp(r.uniform(-17, 10, 3000))
    c = np.array([oracle.round_dtype_c(v, dtype) for v in x])
    assert np.array_equal(c, oracle.round_to_dtype(x, dtype))
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    assert np.array_equal(c, torch.tensor(x, dtype=torch.float64).to(tdt).double().numpy())
    # values already in the dtype are unchanged; halfway cases go to even
    if dtype == "bf16":
        assert oracle.round_dtype_c(1.0 + 2.0 ** -8, "bf16") == 1.0  # tie -> even (1.0)
        assert oracle.round_dtype_c(1.0 + 3 * 2.0 ** -8, "bf16") == 1.0 + 2.0 ** -6
