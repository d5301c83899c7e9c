"""Back-to-back decode-GEMV microbenchmark: each 8B-shape linear of one format
launched `iters` times through the C ABI (msw_linear_decode, PDL launches),
rotating over weight copies that together exceed L2, CUDA events on torch's
stream. The timed launches are replayed from a CUDA graph (no host launch
overhead). `--l2` keeps ONE weight copy (L2-resident when it fits): the
consumer-side (issue) limit rather than HBM. Reports us/launch and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23057_b200._capi import check_engine, engine_lib  # noqa: E402

lib = engine_lib()
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
BYTES = {0: lambda n, k: n * k * 2, 1: lambda n, k: n * k + n * 4, 2: lambda n, k: n * k // 2 + n * k // 64}
l2 = "--l2" in sys.argv
args = [a for a in sys.argv[1:] if not a.startswith("--")]
fmts = [int(f) for f in (args[0] if args else "2,1,0").split(",")]
only = args[1].split(",") if len(args) > 1 else list(SHAPES)
for fmt in fmts:
    for name, (n, k) in SHAPES.items():
        if name not in only:
            continue
        wb = BYTES[fmt](n, k)
        copies = 1 if l2 else max(2, int(300e6 // wb) + 1)
        ws, ss = [], []
        for i in range(copies):
            w = torch.randint(-100, 100, (wb // 4,), dtype=torch.int32, device="cuda")
            ws.append(w)
            if fmt == 1:
                ss.append(torch.rand(n, device="cuda") * 1e-3)
            elif fmt == 2:
                ss.append((torch.rand(n * (k // 128), device="cuda") * 1e-3).half())
            else:
                ss.append(None)
        x = torch.randn(k, device="cuda") * 0.1
        y = torch.empty(n, device="cuda")
        sp = torch.cuda.current_stream().cuda_stream

        def go(i):
            s = ss[i % copies]
            check_engine(lib.msw_linear_decode(fmt, ws[i % copies].data_ptr(),
                                               s.data_ptr() if s is not None else None, n, k,
                                               x.data_ptr(), 1, y.data_ptr(), sp))
        for i in range(10):
            go(i)
        torch.cuda.synchronize()
        iters = 100
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                sp = cs.cuda_stream
                for i in range(iters):
                    go(i)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / iters
        print(f"fmt={fmt} {name:8s} n={n:6d} k={k:6d} {wb / 1e6:8.1f} MB  {us:8.2f} us  "
              f"{wb / us / 1e3:7.0f} GB/s", flush=True)
        del ws, ss
