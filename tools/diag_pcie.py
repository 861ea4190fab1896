#!/usr/bin/env python
"""Pinned host <-> B200 copy bandwidth: H2D alone, D2H alone, both directions at once (two streams),
268 MB each way (the e2e step's volume at 2^24 elements, both parties)."""
import json

import torch


def main():
    n = 2 * (1 << 24)  # int64 elements: both parties' shares of a 2^24 layer
    h_in = torch.empty(n, dtype=torch.int64).pin_memory()
    h_out = torch.empty(n, dtype=torch.int64).pin_memory()
    d_in = torch.empty(n, dtype=torch.int64, device="cuda")
    d_out = torch.empty(n, dtype=torch.int64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = 8 * n

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes_each_way": nbytes, "h2d_GBps": nbytes / t_in / 1e6, "d2h_GBps": nbytes / t_out / 1e6,
                      "duplex_ms": t_both, "duplex_GBps_each_way": nbytes / t_both / 1e6}))


if __name__ == "__main__":
    main()
