"""Edge cases of the boundary: empty / oversize batches (CPU, host-only handle) and a
sequence filling its whole block-table row (GPU)."""
import pytest

from paper_2506_03296_b200 import apex as A
from paper_2506_03296_b200 import build as B
from paper_2506_03296_b200.kvcache import PagedKVCache


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def test_empty_and_oversize_batches_rejected():
    c = PagedKVCache(num_layers=1, num_q_heads=8, num_kv_heads=2, num_blocks=16, max_seqs=8, max_blocks_per_seq=4,
                     max_batch=4, max_new_tokens=64, host_only=True)
    for ids, nn in [([], []), ([0, 1, 2, 3, 4], [1] * 5)]:
        with pytest.raises(A.ApexError) as e:
            c.alloc(ids, nn)
        assert e.value.code == "EINVAL"
    with pytest.raises(A.ApexError) as e:
        c.alloc([0], [65])                      # > max_new_tokens
    assert e.value.code == "EINVAL"
    c.alloc([0], [64])                          # exactly max context = 4 blocks x 16
    assert c.seq_info(0) == (64, [0, 1, 2, 3])
    with pytest.raises(A.ApexError) as e:
        c.alloc([0], [1])                       # would exceed the block-table row
    assert e.value.code == "EINVAL"
    assert c.seq_info(0)[0] == 64


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,hq,hkv", [("bf16", 32, 8), ("f16", 8, 8), ("f32", 4, 4)])
def test_full_block_table_row(cuda_lib, dtype, hq, hkv):
    """A sequence whose context fills every column of its block-table row."""
    import torch

    from helpers import check_close, decode_step, make_cache, oracle_rows, prefill, to_f64
    mbps = 37
    ctx = [mbps * 16, 5, mbps * 16 - 15]
    cache = make_cache(dtype, hq, hkv, num_blocks=3 * mbps, max_seqs=3, max_blocks_per_seq=mbps)
    seqs = [0, 1, 2]
    prefill(cache, seqs, ctx, interleave=100)
    out = decode_step(cache, seqs, ctx)
    torch.cuda.synchronize()
    assert cache.seq_info(0)[0] == mbps * 16
    check_close(to_f64(out, dtype), oracle_rows(seqs, ctx, hq, hkv, dtype), dtype)


@pytest.mark.gpu
def test_failed_alloc_leaves_device_state_usable(cuda_lib):
    """a planner-capacity failure (forced 16-token split over a huge
    step) and a block-exhaustion failure change nothing -- host mirror, device block
    table and lengths stay consistent, so the next step decodes correctly (oracle)."""
    import torch

    from helpers import check_close, decode_step, make_cache, oracle_rows, prefill, to_f64
    ctx = [40, 300, 17]
    seqs = [0, 1, 2]
    cache = make_cache("bf16", 32, 8, num_blocks=6000, max_seqs=8, max_blocks_per_seq=1500, max_batch=8,
                       max_new_tokens=1 << 17)
    prefill(cache, seqs, ctx)
    before = (cache.num_free_blocks(), [cache.seq_info(s) for s in seqs])
    cache.set_split(16)
    with pytest.raises(A.ApexError) as e:        # 5000 blocks fit the pool, but 40000 one-block items
        cache.alloc([3, 4, 5, 6], [20000] * 4)   # exceed the work-list capacity: the planner fails
    assert e.value.code == "EINVAL" and "work items" in str(e.value)
    with pytest.raises(A.ApexError) as e:        # more blocks than the pool has left
        cache.alloc([3, 4, 5, 6, 7], [23000] * 5)
    assert e.value.code == "ENOBLOCKS"
    assert (cache.num_free_blocks(), [cache.seq_info(s) for s in seqs]) == before
    cache.set_split(0)
    out = decode_step(cache, seqs, ctx)
    torch.cuda.synchronize()
    check_close(to_f64(out, "bf16"), oracle_rows(seqs, ctx, 32, 8, "bf16"), "bf16")
