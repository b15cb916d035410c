"""a7 on the GPU: the overlapped all-gather of head-sharded outputs (HeadGather).

Two ranks (processes) each own half of the KV heads and their q-groups for every
request, decode L logical layers over P physical pools, write their heads
head-major into a rotating local buffer, and start the all-gather of layer l
right after its decode so that it overlaps layer l+1 (NCCL when >= 2 GPUs are
visible; otherwise both ranks share GPU 0 and the gather runs over gloo through
pinned host memory on a copy stream + worker thread -- NCCL refuses two ranks on
one device).  Every gathered [Hq][B][D] layer output is compared with the float64
oracle over ALL heads, on the same generated inputs.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CTX = [1, 300, 2000, 4096, 17, 1500]
HQ, HKV, L, P = 32, 8, 4, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2506_03296_b200.kvcache import PagedKVCache, synth_rows, torch_dtype
    from paper_2506_03296_b200.sharding import HeadGather, head_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    kv_lo, kv_hi, q_lo, q_hi = head_range(HKV, HQ, rank, world)
    hq, hkv, B, dt = q_hi - q_lo, kv_hi - kv_lo, len(CTX), "bf16"
    tdt = torch_dtype(dt)
    c = PagedKVCache(num_layers=P, num_q_heads=hq, num_kv_heads=hkv, num_blocks=sum(-(-x // 16) for x in CTX) + 8,
                     max_seqs=B, max_blocks_per_seq=max(-(-x // 16) for x in CTX) + 2, max_batch=B,
                     max_new_tokens=1 << 16, dtype=dt, device=dev)
    seqs = list(range(B))
    pre = {s: x - 1 for s, x in zip(seqs, CTX) if x > 1}
    c.alloc(list(pre), list(pre.values()))
    rb = torch.tensor([s for s in pre for _ in range(pre[s])])
    rp = torch.tensor([t for s in pre for t in range(pre[s])])
    for p in range(P):
        kk = torch.empty((len(rb), hkv, 128), dtype=tdt, device=dev)
        vv = torch.empty_like(kk)
        synth_rows(kk, dt, 1, p, rb, rp, head_offset=kv_lo)
        synth_rows(vv, dt, 2, p, rb, rp, head_offset=kv_lo)
        c.append(p, kk, vv)
    c.alloc(seqs, [1] * B)
    pos, ids = torch.tensor([x - 1 for x in CTX]), torch.tensor(seqs)
    qs, ks, vs = [], [], []
    for p in range(P):
        k1 = torch.empty((B, hkv, 128), dtype=tdt, device=dev)
        v1, q1 = torch.empty_like(k1), torch.empty((B, hq, 128), dtype=tdt, device=dev)
        synth_rows(k1, dt, 1, p, ids, pos, head_offset=kv_lo)
        synth_rows(v1, dt, 2, p, ids, pos, head_offset=kv_lo)
        synth_rows(q1, dt, 0, p, ids, pos, head_offset=q_lo)
        qs.append(q1)
        ks.append(k1)
        vs.append(v1)
    hg = HeadGather(hq, B, 128, tdt, dev, nbuf=2, backend=backend)
    results = []
    for l in range(L):                                  # the bench's per-layer pipeline
        p, j = l % P, l % 2
        if l < P:
            c.append(p, ks[p], vs[p])
        dst = hg.local(j)
        c.decode_into(p, qs[p], [dst], layout="hbd")
        hg.start(j)                                     # overlaps layer l+1's decode
        if l >= 1:                                      # consume layer l-1 one layer late
            prev = hg.result((l - 1) % 2)
            results.append(prev.clone())
            hg.release((l - 1) % 2)
    results.append(hg.result((L - 1) % 2).clone())
    torch.cuda.synchronize()
    hg.close()
    if rank == 0:
        torch.save([r.cpu() for r in results], os.path.join(out_dir, "gathered.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 1])
def test_overlapped_head_gather_matches_oracle(cuda_lib, tmp_path, world):
    """world 2: the sharded pipeline (NCCL with >= 2 GPUs, else gloo on one GPU);
    world 1: the same pipeline through a one-rank NCCL group on CUDA tensors -- NCCL's
    async all_gather_into_tensor, work.wait() and its stream ordering against the decode
    kernels are exercised even where only one GPU is visible."""
    import torch

    from helpers import check_close, oracle_rows
    backend = "nccl" if world == 1 or torch.cuda.device_count() >= 2 else "gloo"
    mp.spawn(_worker, args=(world, _free_port(), backend, str(tmp_path)), nprocs=world, join=True)
    got = torch.load(os.path.join(str(tmp_path), "gathered.pt"))
    assert len(got) == L
    seqs = list(range(len(CTX)))
    for l in range(L):
        assert tuple(got[l].shape) == (HQ, len(CTX), 128)
        ref = oracle_rows(seqs, CTX, HQ, HKV, "bf16", layer=l % P)
        check_close(got[l].permute(1, 0, 2).to(torch.float64).numpy(), ref, "bf16")
