#!/usr/bin/env python
"""Where the pinned-host ReLU pipeline's time goes: the same chunked H2D / D2H stream pattern as
protocol._relu_pair_pinned with and without the kernel, vs one bulk duplex copy."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2309_04875_b200.protocol import _pipeline_chunks  # noqa: E402


def main():
    n = 1 << 24
    h = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(2)]
    o = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(2)]
    d = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(4)]
    s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for chunk in (1 << 20, 1 << 21, 1 << 22):
        def pipe(kernel):
            cur = torch.cuda.current_stream()
            for st in (s_in, s_k, s_out):
                st.wait_stream(cur)
            for lo, hi in _pipeline_chunks(n, chunk):
                with torch.cuda.stream(s_in):
                    d[0][lo:hi].copy_(h[0][lo:hi], non_blocking=True)
                    d[1][lo:hi].copy_(h[1][lo:hi], non_blocking=True)
                s_k.wait_stream(s_in)
                if kernel:
                    with torch.cuda.stream(s_k):
                        d[2][lo:hi].copy_(d[0][lo:hi])
                        d[3][lo:hi].copy_(d[1][lo:hi])
                s_out.wait_stream(s_k)
                with torch.cuda.stream(s_out):
                    o[0][lo:hi].copy_(d[2][lo:hi], non_blocking=True)
                    o[1][lo:hi].copy_(d[3][lo:hi], non_blocking=True)
            s_out.synchronize()

        for kernel in (False, True):
            pipe(kernel)
            t = []
            for _ in range(5):
                t0 = time.perf_counter()
                pipe(kernel)
                t.append(time.perf_counter() - t0)
            res[f"chunk2^{chunk.bit_length() - 1}_{'copy-kernel' if kernel else 'copies-only'}_ms"] = round(1e3 * min(t), 3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
