"""Partitioning of the decode-attention work across the GPUs of one box.

Every (request, kv head) attention is independent, so:
  * request sharding: requests are split across ranks (greedy LPT on context
    length so ragged batches balance their KV bytes); no collective;
  * head sharding: rank r owns kv heads [r*Hkv/N, (r+1)*Hkv/N) and their
    q-groups for every request; the only collective is an all-gather of the
    attention outputs (NCCL over NVLink in production, gloo in CPU tests).
Host logic only; the attention itself runs in libapex.so on each rank.
"""
from __future__ import annotations

import heapq


def lpt_partition(lengths, n_ranks: int):
    """Greedy longest-processing-time assignment of requests to ranks.

    Returns a list (per rank) of request indices, each in ascending order.
    Deterministic: ties broken by request index and rank index."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    heap = [(0, r) for r in range(n_ranks)]
    parts = [[] for _ in range(n_ranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return [sorted(p) for p in parts]


def head_range(num_kv_heads: int, num_q_heads: int, rank: int, world: int):
    """(kv_lo, kv_hi, q_lo, q_hi) owned by `rank` under head sharding."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} kv heads cannot be split over {world} ranks")
    g = num_q_heads // num_kv_heads
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per, rank * per * g, (rank + 1) * per * g


def gather_heads(out_local, group=None, async_op=False):
    """All-gather head-major head-sharded outputs [Hq/N][B][D] -> [Hq][B][D] (NCCL).

    Rank r's slice is rank r's heads, so the gathered tensor is the full head-major
    output with no permute or copy.  With async_op the collective
    is queued behind the current stream's work and (tensor, work) is returned;
    work.wait() makes the *current stream* wait for it (the host is not blocked)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    hl, B, D = out_local.shape
    full = torch.empty((world * hl, B, D), dtype=out_local.dtype, device=out_local.device)
    work = dist.all_gather_into_tensor(full, out_local, group=group, async_op=async_op)
    return (full, work) if async_op else full


class HeadGather:
    """Overlapped all-gather of head-sharded decode outputs.

    Per layer-call: the decode kernel writes this rank's heads head-major into
    ``local(j)`` ([Hq/N][B][D], j = a rotating buffer), ``start(j)`` queues the
    all-gather of that buffer behind the decode on the stream's timeline and returns
    at once, so the next layer's decode (launched right after on the compute stream)
    overlaps the transfer; ``result(j)`` makes the current stream wait for it and
    returns the gathered [Hq][B][D] tensor.  Re-using buffer j (``local(j)``) first
    makes the compute stream wait until the previous gather has read it.

    nccl: ``all_gather_into_tensor(async_op=True)`` on NCCL's internal stream (the
    only collective of the path; NVLink/NVSwitch).  gloo (ranks sharing one GPU, a
    logic test only -- NCCL refuses two ranks per device): the slice is copied to
    pinned host memory on a copy stream, gathered on the CPU by a worker thread over
    a dedicated gloo group (so its collectives never interleave with the main
    thread's), and copied back on the copy stream; the compute stream is not held."""

    def __init__(self, hq_local: int, batch: int, head_dim: int, dtype, device, nbuf: int = 2, group=None,
                 backend: str = "nccl"):
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.backend = backend
        self.nbuf = nbuf
        self.shape = (hq_local, batch, head_dim)
        self._local = [torch.empty(self.shape, dtype=dtype, device=device) for _ in range(nbuf)]
        self._full = [torch.empty((self.world * hq_local, batch, head_dim), dtype=dtype, device=device)
                      for _ in range(nbuf)]
        self._pending = [None] * nbuf
        self._consumed = [None] * nbuf              # consumer reads of the gathered buffer (WAR)
        if backend == "nccl":
            self.group = group
        else:
            import concurrent.futures
            self.group = dist.new_group(backend="gloo")
            self._pool = concurrent.futures.ThreadPoolExecutor(max_workers=1)
            self._copy = torch.cuda.Stream(device)
            self._hloc = [torch.empty(self.shape, dtype=dtype, pin_memory=True) for _ in range(nbuf)]
            self._hfull = [torch.empty(tuple(self._full[0].shape), dtype=dtype, pin_memory=True)
                           for _ in range(nbuf)]
            self._d2h = [torch.cuda.Event() for _ in range(nbuf)]
            self._h2d = [torch.cuda.Event() for _ in range(nbuf)]

    def local(self, j: int):
        """Buffer j for the next decode; the current stream first waits until the
        gather that last read it has (WAR)."""
        import torch
        pend = self._pending[j]
        if pend is not None:
            if self.backend == "nccl":
                pend.wait()
            else:
                torch.cuda.current_stream().wait_event(self._d2h[j])
        return self._local[j]

    def start(self, j: int) -> None:
        import torch
        import torch.distributed as dist
        consumed, self._consumed[j] = self._consumed[j], None
        if self.backend == "nccl":
            if consumed is not None:                      # NCCL's stream waits for the current one
                torch.cuda.current_stream().wait_event(consumed)
            self._pending[j] = dist.all_gather_into_tensor(self._full[j], self._local[j], group=self.group,
                                                           async_op=True)
            return
        if self._pending[j] is not None:
            self._pending[j].result()                     # previous use of buffer j fully done
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream())
        with torch.cuda.stream(self._copy):
            self._copy.wait_event(ready)
            self._hloc[j].copy_(self._local[j], non_blocking=True)
            self._d2h[j].record(self._copy)

        def job():
            self._d2h[j].synchronize()
            dist.all_gather_into_tensor(self._hfull[j], self._hloc[j], group=self.group)
            with torch.cuda.stream(self._copy):
                if consumed is not None:
                    self._copy.wait_event(consumed)
                self._full[j].copy_(self._hfull[j], non_blocking=True)
                self._h2d[j].record(self._copy)
        self._pending[j] = self._pool.submit(job)

    def result(self, j: int):
        """Gathered [Hq][B][D] of buffer j; the current stream waits for the gather."""
        import torch
        pend = self._pending[j]
        if pend is not None:
            if self.backend == "nccl":
                pend.wait()
            else:
                pend.result()
                torch.cuda.current_stream().wait_event(self._h2d[j])
        return self._full[j]

    def release(self, j: int):
        """Called on the stream that consumed result(j): the next gather into buffer j
        waits for that stream's work so far (write-after-read)."""
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._consumed[j] = ev

    def close(self):
        if self.backend != "nccl":
            for p in self._pending:
                if p is not None:
                    p.result()
            self._pool.shutdown()


class SignalledGather:
    """Protocol of the all-gather fused into the decode epilogue.

    Every rank owns, in symmetric memory, ``nbuf`` full head-major output buffers
    [Hq][B][D] and, per buffer, two uint32 arrays ``ready[world]`` and
    ``free[world]``.  For layer-call epoch e (1, 2, ...) on buffer j = e % nbuf, rank r:
      1. waits (``apex_signal_wait``, on its stream) until its own free_j[*] >= the
         epoch buffer j last carried -- every peer has consumed that epoch's rows
         (write-after-read guard);
      2. decodes with ``apex_decode_attention_ex`` into every rank's buffer j at head
         offset r*Hq/N, the kernel's last CTA posting e into slot r of every rank's
         ready_j (system-scope release): no host barrier;
      3. before reading the gathered rows: ``apex_signal_wait(ready_j, world, e)``;
      4. after its consumer is done with them: ``apex_signal_post`` of e into slot r
         of every rank's free_j.
    The pointers are plain device addresses (peer-mapped ones from torch symmetric
    memory on a multi-GPU box; local tensors standing in for peers in the one-GPU
    test), so this class has no torch.distributed dependency itself."""

    def __init__(self, rank: int, world: int, bufs, ready, free, timeout_ns: int = 10_000_000_000):
        """bufs[j][i], ready[j][i], free[j][i]: device pointers of rank i's buffer j /
        ready_j / free_j arrays (as seen from this rank)."""
        self.rank, self.world = rank, world
        self.bufs, self.ready, self.free = bufs, ready, free
        self.nbuf = len(bufs)
        self.timeout_ns = timeout_ns
        self.last_epoch = [0] * self.nbuf

    def decode(self, cache, layer: int, q, epoch: int, hq_total: int, status_ptr: int = 0):
        from . import apex as A
        j = epoch % self.nbuf
        stream = cache._stream()
        if self.last_epoch[j]:
            A.apex_signal_wait(self.free[j][self.rank], self.world, self.last_epoch[j], self.timeout_ns, status_ptr,
                               stream)
        B, D = len(cache.batch_seq_ids), cache.head_dim
        with cache._on_device():
            A.apex_decode_attention_ex(cache.handle, layer, q.data_ptr(), self.bufs[j], D, B * D,
                                       self.rank * cache.num_q_heads, 1.0 / D ** 0.5, stream,
                                       signal_ptrs=self.ready[j], signal_slot=self.rank, signal_value=epoch)
        self.last_epoch[j] = epoch
        return j

    def wait_ready(self, j: int, epoch: int, stream: int, status_ptr: int = 0):
        from . import apex as A
        A.apex_signal_wait(self.ready[j][self.rank], self.world, epoch, self.timeout_ns, status_ptr, stream)

    def release(self, j: int, epoch: int, stream: int):
        from . import apex as A
        A.apex_signal_post(self.free[j], self.rank, epoch, stream)


def symmetric_output(shape, dtype, device, group=None):
    """A full-width output buffer in torch symmetric memory + its rendezvous handle.

    handle.buffer_ptrs holds every rank's (peer-mapped) address of its buffer, to
    be passed as the destinations of apex_decode_attention_ex (SignalledGather).
    NOTE: exercised on one GPU only with local destinations
    (tests/test_fused_gather_gpu.py); the peer-pointer path needs >= 2 GPUs."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(*shape, dtype=dtype, device=device)
    handle = symm_mem.rendezvous(t, group if group is not None else dist.group.WORLD)
    return t, handle
