"""Shared helpers for GPU parity tests: build a paged cache through the C ABI,
prefill it with generator values, run one decode step, and compute the
oracle's answer on the same (regenerated) inputs."""
from __future__ import annotations

import numpy as np

import synth
from synth import TENSOR_K, TENSOR_Q, TENSOR_V

TOL_F32_NORMWISE = 1e-5      # BASELINE.json north_star, reading c6 (row-normwise)
TOL_16BIT_ABS = 2e-2         # BASELINE.json north_star, readings c7/c8


def make_cache(dtype, hq, hkv, num_blocks, max_seqs, max_blocks_per_seq, layers=1, max_batch=None,
               max_new_tokens=1 << 20):
    from paper_2506_03296_b200.kvcache import PagedKVCache
    return PagedKVCache(num_layers=layers, num_q_heads=hq, num_kv_heads=hkv, num_blocks=num_blocks,
                        max_seqs=max_seqs, max_blocks_per_seq=max_blocks_per_seq,
                        max_batch=max_batch or max_seqs, max_new_tokens=max_new_tokens, dtype=dtype)


def gen_dev(cache, tensor, layer, seqs, positions, heads, seed=0, amp=1.0):
    """Device rows [R][heads][D] for (seq, pos) pairs, via the CUDA generator twin."""
    import torch
    from paper_2506_03296_b200.kvcache import synth_rows, torch_dtype
    rb = torch.as_tensor(np.asarray(seqs, dtype=np.int32), device=cache.device)
    rp = torch.as_tensor(np.asarray(positions, dtype=np.int32), device=cache.device)
    out = torch.empty((len(seqs), heads, cache.head_dim), dtype=torch_dtype(cache.dtype), device=cache.device)
    return synth_rows(out, cache.dtype, tensor, layer, rb, rp, seed=seed, amp=amp)


def prefill(cache, seq_ids, ctx, layer=0, seed=0, interleave=0, max_rows=1 << 22, b_ids=None):
    """Write positions 0..ctx[i]-2 of each seq (the decode step appends ctx[i]-1).

    interleave > 0 grows the sequences `interleave` tokens at a time round-robin,
    scattering their physical blocks.  Sequences are prefilled in groups of at
    most max_rows rows.  b_ids maps seq ids to generator request ids (default: same)."""
    if interleave == 0:
        group, rows = [], 0
        for s, c in zip(seq_ids, ctx):
            if group and rows + c - 1 > max_rows:
                prefill(cache, [g for g, _ in group], [c2 for _, c2 in group], layer, seed, -1, max_rows, b_ids)
                group, rows = [], 0
            group.append((s, c))
            rows += c - 1
        if group:
            prefill(cache, [g for g, _ in group], [c2 for _, c2 in group], layer, seed, -1, max_rows, b_ids)
        return
    bid = (lambda s: s) if b_ids is None else (lambda s: b_ids[s])
    todo = {s: c - 1 for s, c in zip(seq_ids, ctx) if c > 1}
    have = {s: 0 for s in todo}
    while todo:
        ids, nn = [], []
        for s in list(todo):
            n = todo[s] if interleave <= 0 else min(interleave, todo[s])
            ids.append(s)
            nn.append(n)
        cache.alloc(ids, nn)
        rows_b, rows_p = [], []
        for s, n in zip(ids, nn):
            rows_b += [bid(s)] * n
            rows_p += list(range(have[s], have[s] + n))
            have[s] += n
            todo[s] -= n
            if todo[s] == 0:
                del todo[s]
        for l in ([layer] if isinstance(layer, int) else layer):
            k = gen_dev(cache, TENSOR_K, l, rows_b, rows_p, cache.num_kv_heads, seed)
            v = gen_dev(cache, TENSOR_V, l, rows_b, rows_p, cache.num_kv_heads, seed)
            cache.append(l, k, v)


def decode_step(cache, seq_ids, ctx, layer=0, seed=0, qamp=1.0, scale=None, fused_append=False):
    """alloc(+1), append the step's token (pos ctx-1), decode; returns out (torch).
    fused_append: one apex_decode_attention_append call instead of append + decode."""
    cache.alloc(list(seq_ids), [1] * len(seq_ids))
    pos = [c - 1 for c in ctx]
    k = gen_dev(cache, TENSOR_K, layer, seq_ids, pos, cache.num_kv_heads, seed)
    v = gen_dev(cache, TENSOR_V, layer, seq_ids, pos, cache.num_kv_heads, seed)
    q = gen_dev(cache, TENSOR_Q, layer, seq_ids, pos, cache.num_q_heads, seed, qamp)
    if fused_append:
        return cache.decode_append(layer, q, k, v, scale=scale)
    cache.append(layer, k, v)
    return cache.decode(layer, q, scale=scale)


def to_f64(out_t, dtype):
    import torch
    return out_t.detach().to(torch.float64).cpu().numpy()


def oracle_rows(seq_ids, ctx, hq, hkv, dtype, layer=0, seed=0, qamp=1.0, rows=None, D=128):
    """float64 oracle for batch rows (all, or `rows` = list of b*hq+h) on regenerated inputs."""
    from oracle import attention as oa
    q = synth.gen_rows(TENSOR_Q, layer, seq_ids, [c - 1 for c in ctx], hq, D, dtype, seed, qamp)
    need = sorted({r // hq for r in rows}) if rows is not None else range(len(seq_ids))
    ks, vs = [], []
    for b in range(len(seq_ids)):
        n = ctx[b] if b in need else 1
        ks.append(synth.gen_seq(TENSOR_K, layer, seq_ids[b], n, hkv, D, dtype, seed))
        vs.append(synth.gen_seq(TENSOR_V, layer, seq_ids[b], n, hkv, D, dtype, seed))
    return oa.decode_attention(q, ks, vs, dtype, rows=rows)


def check_close(got, ref, dtype, tol_f32=TOL_F32_NORMWISE, tol16=TOL_16BIT_ABS):
    """got/ref [..., D] float64.  fp32: row-normwise; 16-bit: elementwise absolute."""
    got = np.asarray(got, dtype=np.float64).reshape(-1, ref.shape[-1])
    ref = np.asarray(ref, dtype=np.float64).reshape(-1, ref.shape[-1])
    assert np.isfinite(got).all(), "non-finite output"
    err = np.abs(got - ref).max(axis=1)
    if dtype == "f32":
        bound = tol_f32 * np.abs(ref).max(axis=1)
        worst = float((err / np.abs(ref).max(axis=1)).max())
        assert (err <= bound).all(), f"fp32 row-normwise error {worst:.3e} > {tol_f32}"
        return worst
    worst = float(err.max())
    assert worst <= tol16, f"16-bit abs error {worst:.3e} > {tol16}"
    return worst
