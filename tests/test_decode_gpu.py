"""GPU parity tests through the C ABI (libapex.so) against the float64 oracle.

Small shapes span several tiles, split items and ragged tails; the BASELINE
configs C1-C5 are covered at full size in test_configs_gpu.py.
"""
import numpy as np
import pytest

import synth
from helpers import check_close, decode_step, gen_dev, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu

# (dtype, Hq, Hkv); Hkv = 1 is a rank's slice under 8-way head sharding of LLaMA-3.1-8B (C5, N = 8: Hq 4, Hkv 1)
COMBOS = [("f32", 4, 4), ("f16", 4, 4), ("f16", 8, 4), ("f16", 8, 2), ("f16", 16, 4), ("f16", 16, 2), ("bf16", 8, 4),
          ("bf16", 16, 4), ("bf16", 16, 2), ("bf16", 4, 1), ("bf16", 8, 1), ("f16", 2, 1)]
RAGGED = [1, 2, 15, 16, 17, 31, 64, 100, 257, 1000, 2049]


def torch_sm_count():
    import torch
    return torch.cuda.get_device_properties(0).multi_processor_count


def run_case(dtype, hq, hkv, ctx, qamp=1.0, split=None, interleave=0, seed=0, num_blocks=None, poison=False,
             sched=None, grid=None):
    import torch
    B = len(ctx)
    mbps = max(-(-c // 16) for c in ctx) + 1
    nb = num_blocks or sum(-(-c // 16) for c in ctx) + 8
    cache = make_cache(dtype, hq, hkv, nb, max_seqs=B + 4, max_blocks_per_seq=mbps)
    if poison:
        for t in cache.kv_pools:
            t.view(torch.uint8).fill_(0xFF)        # NaN bit patterns in every dtype
    if split is not None:
        cache.set_split(split)
    if sched is not None:
        cache.set_sched(sched)
    if grid is not None:
        cache.set_grid(grid)
    seqs = list(range(2, 2 + B))
    prefill(cache, seqs, ctx, seed=seed, interleave=interleave)
    out = decode_step(cache, seqs, ctx, seed=seed, qamp=qamp)
    torch.cuda.synchronize()
    return cache, seqs, to_f64(out, dtype)


def test_generator_twin_bitexact(cuda_lib):
    import torch
    from paper_2506_03296_b200.kvcache import synth_rows, torch_dtype
    rng = np.random.default_rng(0)
    for dtype in ("f32", "f16", "bf16"):
        for (tensor, layer, heads, hoff, amp) in [(0, 0, 32, 0, 1.0), (1, 5, 8, 3, 1.0), (2, 63, 4, 100, 8.0),
                                                   (0, 1, 1, 127, 64.0)]:
            R = 257
            b = rng.integers(0, 65536, R)
            pos = rng.integers(0, 1 << 18, R)
            out = torch.empty((R, heads, 128), dtype=torch_dtype(dtype), device="cuda")
            synth_rows(out, dtype, tensor, layer, torch.as_tensor(b), torch.as_tensor(pos), head_offset=hoff,
                       seed=7, amp=amp)
            host = synth.gen_rows(tensor, layer, b, pos, heads, 128, dtype, seed=7, amp=amp, head_offset=hoff)
            dev = out.cpu()
            dev = dev.numpy() if dtype == "f32" else dev.view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(dev, host), (dtype, tensor)


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
def test_append_bitexact(cuda_lib, dtype):
    import torch
    hkv = 4
    cache = make_cache(dtype, 4 if dtype == "f32" else 8, hkv, num_blocks=40, max_seqs=8, max_blocks_per_seq=16)
    ctx = [3, 40, 17, 100]
    seqs = [0, 3, 5, 6]
    prefill(cache, seqs, ctx, interleave=7)
    # every written slot must hold exactly the generator's row (host scatter check)
    pool_k = cache.k_pools[0].cpu()
    pool_v = cache.v_pools[0].cpu()
    for s, c in zip(seqs, ctx):
        L, blocks = cache.seq_info(s)
        assert L == c - 1
        want_k = synth.gen_seq(1, 0, s, L, hkv, 128, dtype)
        want_v = synth.gen_seq(2, 0, s, L, hkv, 128, dtype)
        for t in range(L):
            blk = blocks[t // 16]
            gk = pool_k[blk, :, t % 16]
            gv = pool_v[blk, :, t % 16]
            if dtype != "f32":
                gk, gv = gk.view(torch.int16).numpy().view(np.uint16), gv.view(torch.int16).numpy().view(np.uint16)
            else:
                gk, gv = gk.numpy(), gv.numpy()
            assert np.array_equal(gk, want_k[t]) and np.array_equal(gv, want_v[t]), (s, t)


@pytest.mark.parametrize("dtype,hq,hkv", COMBOS)
def test_decode_ragged_parity(cuda_lib, dtype, hq, hkv):
    ctx = RAGGED
    _, seqs, out = run_case(dtype, hq, hkv, ctx, interleave=48)
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)
    check_close(out, ref, dtype)


@pytest.mark.parametrize("dtype,hq,hkv", [("f32", 4, 4), ("bf16", 16, 4), ("f16", 4, 4)])
@pytest.mark.parametrize("qamp", [8.0, 64.0])
def test_decode_peaky_scores(cuda_lib, dtype, hq, hkv, qamp):
    ctx = [5, 300, 1111]
    _, seqs, out = run_case(dtype, hq, hkv, ctx, qamp=qamp)
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype, qamp=qamp)
    # reading c6: large logits (q x64) use the looser 1e-4 fp32 normwise bound
    check_close(out, ref, dtype, tol_f32=1e-5 if qamp <= 8 else 1e-4)


@pytest.mark.parametrize("dtype,hq,hkv", COMBOS)
def test_ctx1_returns_v0_bitexact(cuda_lib, dtype, hq, hkv):
    import torch
    _, seqs, out = run_case(dtype, hq, hkv, [1, 1, 1])
    g = hq // hkv
    for i, s in enumerate(seqs):
        v0 = synth.gen_rows(2, 0, [s], [0], hkv, 128, dtype)[0]
        v0 = v0.astype(np.float64) if dtype == "f32" else (
            v0.view(np.float16).astype(np.float64) if dtype == "f16"
            else (v0.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
        for h in range(hq):
            assert np.array_equal(out[i, h], v0[h // g]), (dtype, s, h)


@pytest.mark.parametrize("dtype,hq,hkv", [("f32", 4, 4), ("f16", 4, 4), ("bf16", 16, 4)])
def test_nan_poisoned_pools_do_not_leak(cuda_lib, dtype, hq, hkv):
    ctx = [1, 7, 33, 250]
    _, _, clean = run_case(dtype, hq, hkv, ctx)
    _, _, dirty = run_case(dtype, hq, hkv, ctx, poison=True)
    assert np.isfinite(dirty).all()
    assert np.array_equal(clean, dirty)


@pytest.mark.parametrize("dtype,hq,hkv", [("f32", 4, 4), ("bf16", 16, 4), ("f16", 8, 8)])
def test_block_shuffle_bit_identical(cuda_lib, dtype, hq, hkv):
    ctx = [77, 500, 1025, 3]
    _, _, a = run_case(dtype, hq, hkv, ctx, interleave=0, split=128)
    _, _, b = run_case(dtype, hq, hkv, ctx, interleave=16, split=128, num_blocks=400)
    _, _, c = run_case(dtype, hq, hkv, ctx, interleave=33, split=128, num_blocks=300)
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("dtype,hq,hkv", [("f32", 4, 4), ("bf16", 16, 4), ("f16", 4, 4)])
def test_split_invariance(cuda_lib, dtype, hq, hkv):
    ctx = [1500, 2047, 64]
    outs = [run_case(dtype, hq, hkv, ctx, split=s)[2] for s in (16, 32, 112, 1024, 4096)]
    ref = oracle_rows(list(range(2, 5)), ctx, hq, hkv, dtype)
    for o in outs:
        check_close(o, ref, dtype)
        if dtype == "f32":
            d = np.abs(o - outs[-1]).max(axis=-1) / np.abs(outs[-1]).max(axis=-1)
            assert d.max() <= 1e-6


def test_deterministic_repeat(cuda_lib):
    import torch
    cache = make_cache("bf16", 32, 8, num_blocks=2000, max_seqs=8, max_blocks_per_seq=300)
    ctx = [4000, 123, 2500]
    seqs = [0, 1, 2]
    prefill(cache, seqs, ctx)
    cache.alloc(seqs, [1, 1, 1])
    k = gen_dev(cache, 1, 0, seqs, [c - 1 for c in ctx], 8)
    cache.append(0, k, k)
    q = gen_dev(cache, 0, 0, seqs, [c - 1 for c in ctx], 32)
    outs = [cache.decode(0, q).clone() for _ in range(5)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_errors_and_unsupported(cuda_lib):
    from paper_2506_03296_b200 import apex as A
    cache = make_cache("bf16", 16, 4, num_blocks=8, max_seqs=4, max_blocks_per_seq=4)
    with pytest.raises(A.ApexError) as e:
        A.apex_decode_attention(cache.handle, 0, 0, 0, 0.1)
    assert e.value.code == "EINVAL"          # before any alloc
    cache.alloc([0], [5])
    with pytest.raises(A.ApexError) as e:
        A.apex_kv_append(cache.handle, 3, 16, 16)
    assert e.value.code == "EINVAL"          # bad layer
    with pytest.raises(A.ApexError) as e:
        cache.alloc([1], [16 * 8])
    assert e.value.code in ("ENOBLOCKS", "EINVAL")


@pytest.mark.parametrize("dtype,hq,hkv,batch,ctx", [("f16", 32, 32, 20, 4096), ("bf16", 32, 8, 40, 8192),
                                                   ("f32", 32, 32, 20, 4096)])   # T > 512 P: bandwidth regime
def test_bandwidth_regime_ring_regression(cuda_lib, dtype, hq, hkv, batch, ctx):
    """Regression: with one shared tile ring, a fast consumer warp could pass a
    try_wait.parity on a slot whose previous fill was still in flight (seen as a
    launch failure at C2 sizes).  Repeated decodes of a bandwidth-regime shape."""
    import torch
    from helpers import gen_dev
    cache = make_cache(dtype, hq, hkv, batch * (ctx // 16 + 2), max_seqs=batch, max_blocks_per_seq=ctx // 16 + 2)
    seqs = list(range(batch))
    prefill(cache, seqs, [ctx] * batch)
    out = decode_step(cache, seqs, [ctx] * batch)
    assert cache.decode_launches() == 2
    q = gen_dev(cache, 0, 0, seqs, [ctx - 1] * batch, hq)
    for _ in range(20):
        again = cache.decode(0, q)
        torch.cuda.synchronize()
        assert torch.equal(again, out)
    rows = list(range(0, batch * hq, max(1, batch * hq // 64)))
    ref = oracle_rows(seqs, [ctx] * batch, hq, hkv, dtype, rows=rows)
    check_close(to_f64(out, dtype).reshape(-1, 128)[rows], ref, dtype)


@pytest.mark.parametrize("dtype,hq,hkv", [("bf16", 32, 8), ("f16", 32, 32), ("f32", 8, 8), ("f16", 16, 2)])
@pytest.mark.parametrize("sched", [-1, 0, 1, 100, 1000])
@pytest.mark.parametrize("grid", [7, 0])
def test_streamk_schedules(cuda_lib, dtype, hq, hkv, sched, grid):
    """Stream-K static ranges (+ queue tail) in the bandwidth regime: ragged pairs
    cut at CTA range boundaries are merged like split pairs; parity vs the oracle."""
    ctx = [1000, 3000, 17, 5000, 1, 2500, 4097] if grid == 7 else [80000, 1, 33, 36000, 64000, 48000, 28000, 120001]
    cache, seqs, out = run_case(dtype, hq, hkv, ctx, sched=sched, grid=grid or None, interleave=37, seed=3)
    P = len(cache.plan_ranges()) - 1
    assert P == (7 if grid == 7 else 2 * torch_sm_count())
    T = sum(-(-c // 16) for c in ctx) * hkv
    assert cache.decode_launches() == (2 if T > 512 * P else 1)   # bandwidth regime (+ merge kernel)
    rows = None if grid == 7 else list(range(0, len(ctx) * hq, 3))
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype, seed=3, rows=rows)
    got = out.reshape(-1, 128)[rows] if rows is not None else out
    check_close(got, ref, dtype)


def test_randomized_shapes_and_splits(cuda_lib):
    """Seeded sweep: random dtype/group, ragged lengths, forced or automatic splits."""
    rng = np.random.default_rng(1234)
    combos = COMBOS + [("bf16", 64, 8), ("f16", 32, 4)]
    for case in range(16):
        dtype, hq, hkv = combos[rng.integers(len(combos))]
        ctx = [int(x) for x in rng.integers(1, 3000, size=int(rng.integers(1, 9)))]
        split = [None, 16, 48, 256, 1024][int(rng.integers(5))]
        qamp = float(2 ** int(rng.integers(0, 4)))
        _, seqs, out = run_case(dtype, hq, hkv, ctx, split=split, interleave=int(rng.integers(0, 40)),
                                seed=case, qamp=qamp)
        ref = oracle_rows(seqs, ctx, hq, hkv, dtype, seed=case, qamp=qamp)
        check_close(out, ref, dtype)


def test_continuous_batching_churn(cuda_lib):
    """Serving-style churn: requests finish (apex_kv_release) and new ones arrive
    and reuse freed blocks (which still hold stale K/V) while others keep
    decoding; every step is checked against the oracle on the live batch."""
    import torch
    rng = np.random.default_rng(7)
    hq, hkv, dtype = 16, 4, "bf16"
    cache = make_cache(dtype, hq, hkv, num_blocks=600, max_seqs=32, max_blocks_per_seq=80, max_batch=32)
    live = {}                                   # seq id -> current context length (tokens written)
    next_b = 0
    ids = {}                                    # seq id -> generator request id
    for step in range(12):
        # finish some, admit some
        for s in list(live):
            if rng.random() < 0.25:
                cache.release(s)
                del live[s]
        free_ids = [s for s in range(32) if s not in live]
        for s in free_ids[:int(rng.integers(1, 4))]:
            n0 = int(rng.integers(1, 900))
            ids[s] = next_b
            next_b += 1
            # prefill n0 - 1 tokens of the new request (generator keyed by its request id)
            if n0 > 1:
                cache.alloc([s], [n0 - 1])
                k = gen_dev(cache, 1, 0, [ids[s]] * (n0 - 1), list(range(n0 - 1)), hkv)
                v = gen_dev(cache, 2, 0, [ids[s]] * (n0 - 1), list(range(n0 - 1)), hkv)
                cache.append(0, k, v)
            live[s] = n0 - 1
        seqs = sorted(live)
        cache.alloc(seqs, [1] * len(seqs))
        pos = [live[s] for s in seqs]
        b_ids = [ids[s] for s in seqs]
        k = gen_dev(cache, 1, 0, b_ids, pos, hkv)
        v = gen_dev(cache, 2, 0, b_ids, pos, hkv)
        cache.append(0, k, v)
        q = gen_dev(cache, 0, 0, b_ids, pos, hq)
        out = cache.decode(0, q)
        torch.cuda.synchronize()
        for s in seqs:
            live[s] += 1
        ctx = [live[s] for s in seqs]
        ref = oracle_rows(b_ids, ctx, hq, hkv, dtype)
        check_close(to_f64(out, dtype), ref, dtype)


@pytest.mark.parametrize("dtype,hq,hkv,ctx", [("bf16", 32, 8, [16384]),          # 8 pairs x 37 parts
                                              ("f16", 32, 32, [4096]),           # 32 pairs x 9 parts (8 + 1)
                                              ("bf16", 16, 2, [20000, 3]),       # uneven parts per pair
                                              ("f32", 8, 8, [6000])])
def test_latency_regime_many_part_merge(cuda_lib, dtype, hq, hkv, ctx):
    """Fused (latency-regime) LSE merge of pairs split into many parts (up to ~150):
    the last arriving split merges all partials in-kernel.  Checked against the oracle,
    over two calls (arrival counters re-armed), with the plan asserted to split pairs
    into more than 8 parts.  (A two-level merge tree for these pairs was measured
    slower -- DESIGN.md section 8 -- and not kept.)"""
    import torch
    cache, seqs, out = run_case(dtype, hq, hkv, ctx)
    items, n_merges = cache.plan()
    assert cache.decode_launches() == 1
    parts = {}
    for (b, g, blk0, nblk, part, seq) in items:
        if part >= 0:
            parts[(b, g)] = parts.get((b, g), 0) + 1
    assert parts and max(parts.values()) > 8, parts
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)
    check_close(out, ref, dtype)
    q = gen_dev(cache, 0, 0, seqs, [c - 1 for c in ctx], hq)
    again = cache.decode(0, q)
    torch.cuda.synchronize()
    assert np.array_equal(to_f64(again, dtype), out)          # deterministic, counters re-armed
