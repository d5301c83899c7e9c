import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "oracle"))
import numpy as np, torch
import oracle as O
from paper_2605_23057_b200._capi import check_engine, engine_lib
for (n, k, t) in [(256, 14336, 6), (256, 14336, 5), (256, 12288, 6), (512, 4096, 6)]:
    w = O.fill_fp16(n, k, 11, 1234 + n, 7)
    x = np.random.default_rng(1).standard_normal((t, k)).astype(np.float32)
    dw = torch.from_numpy(w.view(np.int16)).cuda(); dx = torch.from_numpy(x).cuda()
    dy = torch.empty((t, n), device="cuda")
    check_engine(engine_lib().msw_linear(0, dw.data_ptr(), None, n, k, dx.data_ptr(), t, dy.data_ptr(), None))
    torch.cuda.synchronize()
    y = dy.cpu().numpy(); ref = O.linear(0, w, None, x)
    err = np.abs(y - ref) / np.abs(ref).max()
    bad = np.argwhere(err > 1e-4)
    print(n, k, t, "maxerr", err.max(), "bad count", len(bad), "bad rows(tok)", sorted(set(bad[:, 0].tolist()))[:8], "bad cols", sorted(set((bad[:, 1] % 16).tolist()))[:16], "tiles", sorted(set((bad[:, 1] // 16).tolist()))[:8])
