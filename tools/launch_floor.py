"""Event-timed floor of one tiny launch on this GPU (L2 flushed like the latency probe).

    python tools/launch_floor.py
Prints the median us between two CUDA events around a 1-element tensor.zero_()
(the stream/launch overhead any single-kernel decode call pays in its event time).
"""
import json
import statistics

import torch


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    x = torch.empty(1, device="cuda")
    res = {}
    for name, flushed in (("flushed", True), ("warm", False)):
        times = []
        for r in range(23):
            if flushed:
                flush.fill_(r & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x.zero_()
            e1.record()
            torch.cuda.synchronize()
            if r >= 3:
                times.append(e0.elapsed_time(e1) * 1e3)
        res[name] = {"us_median": round(statistics.median(times), 2), "us_min": round(min(times), 2)}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e1.record()
    torch.cuda.synchronize()
    res["empty_event_pair_us"] = round(e0.elapsed_time(e1) * 1e3, 2)
    print(json.dumps({"launch_floor": res}))
    # streaming floor: a plain torch reduction over N bytes of bf16 (read-only), L2 flushed by
    # reading (clean) or writing (dirty) a 512 MiB buffer first
    sink = torch.zeros((), dtype=torch.int64, device="cuda")
    for nbytes in (16 << 20, 64 << 20, 128 << 20, 256 << 20, 512 << 20, 4 << 30):
        src = torch.ones(nbytes // 2, dtype=torch.bfloat16, device="cuda")
        for mode in ("read", "write"):
            times = []
            for r in range(13):
                if mode == "write":
                    flush.fill_(r & 0xff)
                else:
                    sink.copy_(flush.view(torch.int64).sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                src.sum(dtype=torch.float32)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    times.append(e0.elapsed_time(e1) * 1e3)
            us = statistics.median(times)
            print(json.dumps({"stream_floor": {"bytes": nbytes, "flush": mode, "us": round(us, 2),
                                               "gbs": round(nbytes / us / 1e3, 1)}}), flush=True)
        del src


if __name__ == "__main__":
    main()
