"""Out-of-bounds write checks of the whole step, without compute-sanitizer.

compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing a
reset), so the writes of every kernel a step launches are checked with canaries
instead, on the paths the sanitizer test covered (split items + merge kernel,
latency-regime fused merge, fused append, strided multi-destination epilogue):

* pools: every byte is poisoned (0xFF) first; after prefill + append + decode
  exactly the slots [0, len) of each sequence's blocks hold generator rows and
  every other byte of every pool -- unowned blocks, slots past len, other layers
  -- is still 0xFF (append, fused append and the block-table delta kernel write
  nowhere else; decode and merge write no pool byte);
* outputs: the output is a view inside a larger sentinel-filled buffer; rows
  before and after it, and (strided epilogue) the heads of other ranks, keep
  their sentinel bits, while every owned element is finite and matches the oracle;
* the block table and lengths on the device equal the host allocator's view.
"""
import numpy as np
import pytest

from helpers import check_close, gen_dev, make_cache, oracle_rows, prefill, to_f64

pytestmark = pytest.mark.gpu

CASES = [("bf16", 16, 4, 64, False), ("bf16", 32, 8, None, True), ("f16", 4, 4, None, False),
         ("f16", 32, 32, 32, True), ("f32", 4, 4, 32, False), ("f32", 8, 8, None, True)]


def _owned_mask(cache, seqs, n_blocks, layer_pool):
    """bool [num_blocks][16]: slots holding tokens of a live sequence."""
    mask = np.zeros((n_blocks, 16), dtype=bool)
    for s in seqs:
        ln, blocks = cache.seq_info(s)
        for i, blk in enumerate(blocks):
            n = min(16, ln - 16 * i)
            if n > 0:
                mask[blk, :n] = True
    return mask


@pytest.mark.parametrize("dtype,hq,hkv,split,fused", CASES)
def test_step_writes_stay_in_bounds(cuda_lib, dtype, hq, hkv, split, fused):
    import torch

    from paper_2506_03296_b200.kvcache import torch_dtype
    ctx = [1, 100, 257, 33]
    seqs = [0, 1, 3, 5]                        # non-contiguous seq ids: table rows 2 and 4 stay empty
    nb = 96
    cache = make_cache(dtype, hq, hkv, nb, max_seqs=8, max_blocks_per_seq=24, layers=2)
    if split:
        cache.set_split(split)
    for t in cache.kv_pools:
        t.view(torch.uint8).fill_(0xFF)
    prefill(cache, seqs, ctx, layer=1)
    cache.alloc(seqs, [1] * len(seqs))
    pos = [c - 1 for c in ctx]
    k = gen_dev(cache, 1, 1, seqs, pos, hkv)
    v = gen_dev(cache, 2, 1, seqs, pos, hkv)
    q = gen_dev(cache, 0, 1, seqs, pos, hq)
    B, D, tdt = len(seqs), 128, torch_dtype(dtype)
    big = torch.empty((B + 2, hq, D), dtype=tdt, device=cache.device)
    big.view(torch.uint8).fill_(0xA5)
    sentinel = big[0].clone()
    out = big[1:B + 1]
    if fused:
        cache.decode_append(1, q, k, v, out=out)
    else:
        cache.append(1, k, v)
        cache.decode(1, q, out=out)
    torch.cuda.synchronize()
    # outputs: neighbours untouched, owned rows correct
    assert torch.equal(big[0].view(torch.uint8), sentinel.view(torch.uint8))
    assert torch.equal(big[B + 1].view(torch.uint8), sentinel.view(torch.uint8))
    check_close(to_f64(out, dtype), oracle_rows(seqs, ctx, hq, hkv, dtype, layer=1), dtype)
    # pools: layer 0 never written; layer 1 written exactly on owned slots
    assert bool((cache.kv_pools[0].view(torch.uint8) == 0xFF).all()), "write into an unused layer's pool"
    mask = _owned_mask(cache, seqs, nb, 1)
    pool = cache.kv_pools[1].view(torch.uint8).cpu().numpy()      # [nb][Hkv][2][16][D*es]
    untouched = (pool == 0xFF).all(axis=-1)                       # [nb][Hkv][2][16]
    owned = np.broadcast_to(mask[:, None, None, :], untouched.shape)
    assert untouched[~owned].all(), "a pool slot outside [0, len) of a live sequence was written"
    assert not untouched[owned].any(), "an owned slot was never written"
    # device block table / lengths == the host allocator
    bt = cache.block_table.cpu().numpy()
    lens = cache.seq_lens.cpu().numpy()
    for s in seqs:
        ln, blocks = cache.seq_info(s)
        assert lens[s] == ln and list(bt[s, :len(blocks)]) == blocks
    cache.close()


@pytest.mark.parametrize("layout", ["bhd", "hbd"])
@pytest.mark.parametrize("split", [None, 32])
def test_strided_epilogue_writes_only_its_heads(cuda_lib, layout, split):
    """apex_decode_attention_ex into two destinations at head offset 8 of a 32-head
    buffer (a rank's slice under 4-way head sharding): every other head and the rows
    around the buffers keep their sentinel bits, in both output layouts."""
    import torch

    from paper_2506_03296_b200.kvcache import torch_dtype
    dtype, hq, hkv, H, off = "bf16", 8, 2, 32, 8
    ctx = [5, 700, 64]
    seqs = [0, 1, 2]
    cache = make_cache(dtype, hq, hkv, 96, max_seqs=4, max_blocks_per_seq=48)
    if split:
        cache.set_split(split)
    prefill(cache, seqs, ctx)
    cache.alloc(seqs, [1] * 3)
    pos = [c - 1 for c in ctx]
    cache.append(0, gen_dev(cache, 1, 0, seqs, pos, hkv), gen_dev(cache, 2, 0, seqs, pos, hkv))
    q = gen_dev(cache, 0, 0, seqs, pos, hq)
    B, D, tdt = 3, 128, torch_dtype(dtype)
    shape = (B, H, D) if layout == "bhd" else (H, B, D)
    n = int(np.prod(shape))
    bigs = [torch.empty((n + 2 * 4096,), dtype=tdt, device=cache.device) for _ in range(2)]
    for t in bigs:
        t.view(torch.uint8).fill_(0x5A)
    dsts = [t[4096:4096 + n].view(shape) for t in bigs]
    cache.decode_into(0, q, dsts, head_offset=off, layout=layout)
    torch.cuda.synchronize()
    ref = oracle_rows(seqs, ctx, hq, hkv, dtype)                  # [B][hq][D]
    for t, d in zip(bigs, dsts):
        raw = t.view(torch.int16).cpu().numpy()
        fill = np.int16(0x5A5A)
        assert (raw[:4096] == fill).all() and (raw[4096 + n:] == fill).all(), "write outside the buffer"
        bhd = d if layout == "bhd" else d.permute(1, 0, 2)
        keep = torch.ones(H, dtype=torch.bool)
        keep[off:off + hq] = False
        others = bhd[:, keep].contiguous().view(torch.int16).cpu().numpy()
        assert (others == fill).all(), "write into another rank's heads"
        check_close(to_f64(bhd[:, off:off + hq].contiguous(), dtype), ref, dtype)
    cache.close()
