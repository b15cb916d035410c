"""Asynchronous-Overlap analogue on one B200 (§3.3).

APEX runs the attention of CPU-designated requests concurrently with the GPU's
work and synchronises each layer's offloaded result only when the next
iteration needs it ("deferred synchronization"); before that point
the GPU checks whether the result is ready and, if it is not, carries on and
re-checks in the next iteration instead of stalling.  On a B200 the
"CPU lane" becomes a second CUDA stream with its own paged cache and handle:

* ``launch(layer, q, k_new, v_new)`` enqueues, on the lane's stream and after
  the caller's stream has produced q/k/v (event wait, no host sync), the
  append + decode attention of the offloaded requests for that layer into a
  per-layer output buffer, and records a per-layer completion event;
* ``ready(layer)`` is a non-blocking readiness check (``cudaEventQuery``);
* ``collect(layer)`` returns the layer's output with the caller's stream made
  to wait for it if it is ready, else ``None`` -- the caller proceeds and
  re-checks later (P:311's non-stalling re-check).

No compute happens here: append/decode are the C ABI calls of the lane's
``PagedKVCache``.  Measured on B200 (``tools/overlap_b200.py``,
``profiles/apex_overlap_b200.json``): both lanes draw on the same HBM, so the
overlap does not pay there; the mechanism is kept for
heterogeneous lanes and tested for parity and non-stalling behaviour.
"""
from __future__ import annotations


class DeferredLane:
    def __init__(self, cache, num_layers: int):
        """cache: the lane's PagedKVCache (its own requests, pools and handle)."""
        import torch
        self.cache = cache
        self.stream = torch.cuda.Stream(cache.device)
        self.outs = [None] * num_layers
        self.done = [None] * num_layers
        self.pending = [False] * num_layers

    def alloc(self, seq_ids, n_new):
        """Reserve this iteration's slots on the lane's stream (the lane's plan)."""
        import torch
        with torch.cuda.stream(self.stream):
            self.cache.alloc(seq_ids, n_new)

    def launch(self, layer: int, q, k_new, v_new, phys_layer: int | None = None):
        import torch
        p = layer if phys_layer is None else phys_layer
        produced = torch.cuda.Event()
        produced.record(torch.cuda.current_stream(self.cache.device))
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(produced)
            if self.outs[layer] is None or self.outs[layer].shape != q.shape:
                self.outs[layer] = torch.empty_like(q)
            self.cache.append(p, k_new, v_new)
            self.cache.decode(p, q, out=self.outs[layer])
            ev = torch.cuda.Event()
            ev.record(self.stream)
        # the inputs must outlive the lane's use of them
        q.record_stream(self.stream)
        k_new.record_stream(self.stream)
        v_new.record_stream(self.stream)
        self.done[layer] = ev
        self.pending[layer] = True

    def ready(self, layer: int) -> bool:
        ev = self.done[layer]
        return ev is not None and ev.query()

    def collect(self, layer: int):
        """The layer's output if it is complete (the caller's stream is ordered after
        it), else None without blocking."""
        import torch
        if not self.pending[layer] or not self.ready(layer):
            return None
        torch.cuda.current_stream(self.cache.device).wait_event(self.done[layer])
        self.pending[layer] = False
        return self.outs[layer]
