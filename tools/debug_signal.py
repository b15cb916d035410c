"""Debug aid: one fused-merge (latency regime) decode with completion signals; prints the
signal arrays, the wait status and the per-layer signal counter afterwards."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from helpers import make_cache, prefill, gen_dev
    from paper_2506_03296_b200 import apex as A
    for split in (0, 64):
        ctx = [1, 300, 2000, 4096, 17]
        B = len(ctx)
        c = make_cache("bf16", 16, 4, sum(-(-x // 16) for x in ctx) + 4, max_seqs=B,
                       max_blocks_per_seq=max(-(-x // 16) for x in ctx) + 1)
        c.set_split(split)
        seqs = list(range(B))
        prefill(c, seqs, ctx)
        c.alloc(seqs, [1] * B)
        k = gen_dev(c, 1, 0, seqs, [x - 1 for x in ctx], 4)
        c.append(0, k, k)
        q = gen_dev(c, 0, 0, seqs, [x - 1 for x in ctx], 16)
        out = torch.full((16, B, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
        sig = torch.zeros(4, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        s = torch.cuda.current_stream().cuda_stream
        A.apex_decode_attention_ex(c.handle, 0, q.data_ptr(), [out.data_ptr()], 128, B * 128, 0, 0.088, s,
                                   signal_ptrs=[sig.data_ptr()], signal_slot=1, signal_value=5)
        torch.cuda.synchronize()
        ws = c.workspace.view(torch.int32)
        print("split", split, "launches", c.decode_launches(), "sig", sig.tolist(), "counters",
              ws[:4].tolist(), "sigctr", ws[128:130].tolist(), "nan", bool(out.isnan().any()), flush=True)


if __name__ == "__main__":
    main()
