"""Debug aid: the two-'rank' signalled gather of tests/test_fused_gather_gpu.py with
per-wait status words, short timeouts and variants (reader queued first / after)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from test_fused_gather_gpu import _rank_cache
    from paper_2506_03296_b200 import apex as A
    dtype, hq, hkv, world = "bf16", 32, 8, 2
    ctx = [1, 300, 2000, 4096, 17]
    seqs, B = list(range(len(ctx))), len(ctx)
    for split in (0, 64):
        for reader_first in (False, True):
            caches, qs = [], []
            for r in range(world):
                c, (q,) = _rank_cache(dtype, hq, hkv, world, r, ctx, seqs)
                c.set_split(split)
                c.alloc(seqs, [0] * B)
                caches.append(c)
                qs.append(q)
            bufs = [torch.full((hq, B, 128), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
            sig = [torch.zeros((2, world), dtype=torch.int32, device="cuda") for _ in range(world)]
            st = torch.zeros(8, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            reader, writer = torch.cuda.Stream(), torch.cuda.Stream()

            def rd():
                for r in range(world):
                    A.apex_signal_wait(sig[r].data_ptr(), world, 1, 2_000_000_000, st.data_ptr() + 4 * r,
                                       reader.cuda_stream)

            def wr():
                with torch.cuda.stream(writer):
                    for r in range(world):
                        c = caches[r]
                        A.apex_decode_attention_ex(c.handle, 0, qs[r].data_ptr(), [b.data_ptr() for b in bufs], 128,
                                                   B * 128, r * 16, 0.088, writer.cuda_stream,
                                                   signal_ptrs=[s.data_ptr() for s in sig], signal_slot=r,
                                                   signal_value=1)
            t0 = time.time()
            if reader_first:
                rd()
                wr()
            else:
                wr()
                torch.cuda.synchronize()
                rd()
            torch.cuda.synchronize()
            ws = [c.workspace.view(torch.int32)[128:130].tolist() for c in caches]
            print(f"split {split} reader_first {reader_first}: {time.time() - t0:.2f}s status {st[:2].tolist()} "
                  f"sig {[s.tolist() for s in sig]} sigctr {ws} nan {[bool(b.isnan().any()) for b in bufs]} "
                  f"launches {caches[0].decode_launches()}", flush=True)


if __name__ == "__main__":
    main()
