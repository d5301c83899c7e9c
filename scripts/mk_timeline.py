"""Phase timeline of the persistent decode step (diagnostics build
libmsw_engine_trace.so with -DMSW_TRACE): per grid phase, when the last CTA's
consumers got past the input barrier, and when the epilogue arrivals of the
GEMV phases landed (max over CTAs), relative to the kernel start, in us."""
import ctypes as C
import os
import sys

os.environ["MSW_ENGINE_SO"] = "libmsw_engine_trace.so"
os.environ["MSW_MK"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23057_b200 import engine_cfg  # noqa: E402
from paper_2605_23057_b200._capi import engine_lib  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
target = sys.argv[2] if len(sys.argv) > 2 else "llama8b"
lib = engine_lib()
eng = Engine(engine_cfg(target=target, draft=None, modes=[mode], kv_blocks=128, max_seq_len=512))
p = np.arange(128, dtype=np.int32) % 1000
eng.run(mode, p, 8)
buf = torch.zeros(148 * 8192, dtype=torch.int64, device="cuda")
assert lib.msw_mk_trace_set(C.c_void_p(buf.data_ptr())) == 0
eng.run(mode, p, 3)  # prefill + 2 decode steps; the buffer keeps the last step
torch.cuda.synchronize()
lib.msw_mk_trace_set(C.c_void_p(0))
t = buf.cpu().numpy().reshape(148, 8192)
t0 = t[:, 1000][t[:, 1000] > 0].min()
rel = lambda a: (a - t0) / 1000.0
nb = 2 + 5 * 32
kinds = ["qkv", "attn", "o", "gu", "down"]
print(f"mode {mode}: embed done (max over CTAs) {rel(t[:, 1000].max()):.2f} us")
prev, deltas = 0.0, {k: [] for k in kinds + ["head"]}
for j in range(nb - 1):
    w = t[:, j]
    w = w[w > 0]
    if not len(w):
        continue
    kind = kinds[j % 5] if j < nb - 2 else "head"
    passed = rel(w.max())
    if j < 12 or j > nb - 4:
        print(f"wait {j:3d} before {kind:5s}: consumers past barrier first {rel(w.min()):8.2f} "
              f"last {passed:8.2f} us (+{passed - prev:6.2f})")
    deltas[kind].append(passed - prev)
    prev = passed
# the phase that ENDS at wait j is the one before it
print("mean time from the previous barrier to this one, by the phase that ran in between:")
order = ["down", "qkv", "attn", "o", "gu"]
for k, prevk in zip(kinds, order):
    print(f"  {prevk:5s} -> {k:5s}: {np.mean(deltas[k][1:]):7.2f} us")
at = t[:, 900:932]
print("attention done (max over CTAs) per layer, first 6:", np.round(rel(at.max(axis=0)), 1)[:6])
pr = t[:, 600:600 + 4 * 32 + 1]
print("producer phase start (median over CTAs) first 12:", np.round(rel(np.median(pr, axis=0)), 1)[:12])
ea = t[:, 300:300 + 4 * 32 + 1]
print("epilogue arrivals (max over CTAs) first 12:", np.round(rel(ea.max(axis=0)), 1)[:12])
if t[0, 8002] > 0:
    print(f"SM clock over the step (CTA 0): {(t[0, 8003] - t[0, 8001]) / (t[0, 8002] - t[0, 8000]) * 1000:.0f} MHz, "
          f"step {(t[0, 8002] - t[0, 8000]) / 1000:.1f} us")
print("CTA 0, layer 5: pass / prologue-done per GEMV phase:",
      [(round(float(rel(t[0, j])), 2), round(float(rel(t[0, 4096 + j])), 2)) for j in (25, 27, 28, 29)])
pr = t[0, 5000:5000 + 5 * 130].reshape(130, 5)
print("CTA 0 prologue internals (us from prologue start): x-arrived, reduced, converted, synced")
for c in range(20, 25):
    r0 = pr[c]
    if r0[0] > 0:
        print("   call", c, [round((v - r0[0]) / 1000, 2) if v > 0 else None for v in r0[1:]])
# phase anatomy, layer 5 (barriers 25..29), CTA 0 and the max over CTAs
def row(j):
    return t[:, j]
print("layer 5 anatomy (us): phase | last CTA past barrier | prologue done (CTA0, max) | epilogue arrival (max) ")
gem = {25: 20, 27: 21, 28: 22, 29: 23}  # barrier index -> epilogue arrival slot (4 per layer + l*4)
for j, kind in zip(range(25, 30), ["qkv", "attn", "o", "gu", "down"]):
    passed = rel(row(j)[row(j) > 0].max())
    pro = t[:, 4096 + j]
    pro_s = f"{rel(pro[0]):8.2f} {rel(pro[pro > 0].max()):8.2f}" if (pro > 0).any() else "   -        -   "
    print(f"  {kind:5s} {passed:8.2f}   {pro_s}")
for l in (5,):
    ea = t[:, 300 + 4 * l: 300 + 4 * l + 4]
    print("  epilogue arrivals qkv/o/gu/down (max over CTAs):", np.round(rel(ea.max(axis=0)), 2))
    print("  attention done (max):", round(float(rel(t[:, 900 + l].max())), 2))
for cta in (0, 70):
    pi = rel(t[cta, 1024:2048]); ci = rel(t[cta, 2048:3072]); et = rel(t[cta, 3072:4096])
    n = int((t[cta, 1024:2048] > 0).sum()); m = int((t[cta, 3072:4096] > 0).sum())
    print(f"CTA {cta}: {n} stages, {m} tiles")
    print("  stage: issued / consumed (warp 0), first 40:")
    for s0 in range(0, min(n, 40)):
        print(f"    {s0:3d} {pi[s0]:8.2f} {ci[s0]:8.2f}  lat {ci[s0] - pi[s0]:6.2f}")
    print("  epilogue tile done, first 30:", np.round(et[:min(m, 30)], 2))
eng.close()
