"""f3 across processes: the fused all-gather epilogue with completion flags, where the
destinations of a rank's stores are ANOTHER PROCESS's buffers mapped through CUDA IPC.

Two ranks (processes on one GPU) each own half of the KV heads.  Each allocates its
full-width head-major output buffer [Hq][B][D] and a [2][world] ready/free flag array,
and hands both to the other rank as CUDA IPC mappings (torch.multiprocessing).  Per
epoch, each rank's decode (apex_decode_attention_ex) stores its head slice into both
ranks' buffers and its last CTA posts the epoch into both ranks' ready flags
(system-scope release); each rank's reader stream, queued BEFORE the writers, waits on
its own flags (apex_signal_wait, acquire), snapshots its buffer and posts "consumed"
into both ranks' free flags, which gate the next epoch's writes (write-after-read).
Epoch 2 decodes another layer (other data), so stale rows cannot pass.  This is the
SignalledGather protocol of sharding.py with out-of-process pointers -- the closest a
one-GPU box gets to NVLink peer pointers (which it cannot map).  Snapshots vs the
float64 oracle over all heads.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CTX = [1, 300, 2000, 4096, 17]
HQ, HKV, WORLD, EPOCHS = 32, 8, 2, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, queues, out_dir, split):
    import torch
    import torch.distributed as dist

    from paper_2506_03296_b200.kvcache import PagedKVCache, synth_rows, torch_dtype
    from paper_2506_03296_b200.sharding import SignalledGather, head_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    kv_lo, kv_hi, q_lo, q_hi = head_range(HKV, HQ, rank, WORLD)
    hq, hkv, B, dt = q_hi - q_lo, kv_hi - kv_lo, len(CTX), "bf16"
    tdt = torch_dtype(dt)
    c = PagedKVCache(num_layers=EPOCHS, num_q_heads=hq, num_kv_heads=hkv,
                     num_blocks=sum(-(-x // 16) for x in CTX) + 8, max_seqs=B,
                     max_blocks_per_seq=max(-(-x // 16) for x in CTX) + 2, max_batch=B, max_new_tokens=1 << 16,
                     dtype=dt, device="cuda")
    c.set_split(split)
    seqs = list(range(B))
    pre = {s: x - 1 for s, x in zip(seqs, CTX) if x > 1}
    c.alloc(list(pre), list(pre.values()))
    rb = torch.tensor([s for s in pre for _ in range(pre[s])])
    rp = torch.tensor([t for s in pre for t in range(pre[s])])
    for l in range(EPOCHS):
        kk = torch.empty((len(rb), hkv, 128), dtype=tdt, device="cuda")
        vv = torch.empty_like(kk)
        synth_rows(kk, dt, 1, l, rb, rp, head_offset=kv_lo)
        synth_rows(vv, dt, 2, l, rb, rp, head_offset=kv_lo)
        c.append(l, kk, vv)
    c.alloc(seqs, [1] * B)
    pos, ids = torch.tensor([x - 1 for x in CTX]), torch.tensor(seqs)
    qs = []
    for l in range(EPOCHS):
        k1 = torch.empty((B, hkv, 128), dtype=tdt, device="cuda")
        v1, q1 = torch.empty_like(k1), torch.empty((B, hq, 128), dtype=tdt, device="cuda")
        synth_rows(k1, dt, 1, l, ids, pos, head_offset=kv_lo)
        synth_rows(v1, dt, 2, l, ids, pos, head_offset=kv_lo)
        synth_rows(q1, dt, 0, l, ids, pos, head_offset=q_lo)
        c.append(l, k1, v1)
        qs.append(q1)
    # own buffer + flags; the peer's arrive as CUDA IPC mappings
    buf = torch.full((HQ, B, 128), float("nan"), dtype=tdt, device="cuda")
    sig = torch.zeros((2, WORLD), dtype=torch.int32, device="cuda")         # [ready; free]
    torch.cuda.synchronize()
    queues[1 - rank].put((buf, sig))
    peer_buf, peer_sig = queues[rank].get()
    bufs, sigs = [None] * WORLD, [None] * WORLD
    bufs[rank], sigs[rank], bufs[1 - rank], sigs[1 - rank] = buf, sig, peer_buf, peer_sig
    sg = SignalledGather(rank, WORLD, [[b.data_ptr() for b in bufs]], [[s.data_ptr() for s in sigs]],
                         [[s.data_ptr() + 4 * WORLD for s in sigs]])
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    reader, writer = torch.cuda.Stream(), torch.cuda.Stream()
    buf.clone()                                          # load the copy kernel before anything spins (lazy
    torch.cuda.synchronize()                             # loading would block behind the spinning wait)
    dist.barrier()                                       # both ranks hold both mappings
    snaps = []
    for epoch in range(1, EPOCHS + 1):
        with torch.cuda.stream(reader):                  # queued first: spins until both ranks' flags land
            sg.wait_ready(0, epoch, reader.cuda_stream, status.data_ptr())
            snaps.append(buf.clone())
            sg.release(0, epoch, reader.cuda_stream)
        with torch.cuda.stream(writer):                  # epoch e >= 2 waits on the free flags first
            sg.decode(c, epoch - 1, qs[epoch - 1], epoch, HQ, status.data_ptr())
        torch.cuda.synchronize()
    dist.barrier()                                       # the peer's last posts into this rank's flags landed
    flags = sig.tolist()
    torch.save({"snaps": [s.cpu() for s in snaps], "status": int(status.item()), "flags": flags},
               os.path.join(out_dir, f"rank{rank}.pt"))
    dist.barrier()                                       # the peer is done with this rank's mappings
    dist.destroy_process_group()


@pytest.mark.parametrize("split", [0, 64])
def test_fused_gather_across_processes_ipc(cuda_lib, tmp_path, split):
    import torch

    from helpers import check_close, oracle_rows
    ctx = mp.get_context("spawn")
    queues = [ctx.Queue(), ctx.Queue()]
    mp.spawn(_worker, args=(_free_port(), queues, str(tmp_path), split), nprocs=WORLD, join=True)
    seqs = list(range(len(CTX)))
    refs = [oracle_rows(seqs, CTX, HQ, HKV, "bf16", layer=l) for l in range(EPOCHS)]
    for r in range(WORLD):
        res = torch.load(os.path.join(str(tmp_path), f"rank{r}.pt"))
        assert res["status"] == 0, f"rank {r}: a flag wait timed out"
        assert res["flags"] == [[EPOCHS] * WORLD, [EPOCHS] * WORLD]
        for l, snap in enumerate(res["snaps"]):
            check_close(snap.permute(1, 0, 2).to(torch.float64).numpy(), refs[l], "bf16")
