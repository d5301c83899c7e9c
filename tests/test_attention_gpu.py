"""Decode / continuous-batching attention (attn_decode_kernel) at the 8B
shape (32 q heads, 8 kv heads, head_dim 128, GQA group 4) and long contexts,
against a float64 numpy reference of the same op, through the C ABI entry
msw_attention_decode. Covers the split-KV path with the in-kernel merge at
4K-8K positions (nsplit up to 32: BASELINE config 5's 8K requests), ragged
tokens of different sequences in one launch (continuous batching), shuffled
physical blocks, and the fused RoPE + KV append of the newest position.

Reference: RoPE rotate-half on q and the new k with the given cos/sin table,
q / k / v rounded to fp16, scores q.k/sqrt(D), softmax, weighted sum of v.
Bar: max |gpu - ref| / max |ref| < 2e-3 (fp16 P in the tensor-core tile)."""
import numpy as np
import pytest

from paper_2605_23057_b200._capi import check_engine, engine_lib

pytestmark = pytest.mark.gpu

HQ, HK, D = 32, 8, 128


def _rope_table(max_pos, d, theta=500000.0):
    inv = theta ** (-(np.arange(d // 2, dtype=np.float64) * 2.0) / d)
    ang = (np.arange(max_pos, dtype=np.float32)[:, None] * inv.astype(np.float32)[None, :]).astype(np.float32)
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)  # [max_pos, d/2, 2]


def _rope(x, cs):
    h = x.shape[-1] // 2
    c, s = cs[:, 0].astype(np.float64), cs[:, 1].astype(np.float64)
    x0, x1 = x[..., :h], x[..., h:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)


def _f16(a):
    return a.astype(np.float16).astype(np.float64)


@pytest.mark.parametrize("ctxs,nsplit", [([8000], 32), ([4100], 5), ([300, 5000, 8191], 16),
                                         ([1], 32), ([17, 33], 1)])
def test_attention_decode_long_context_8b_shape(cuda_ok, ctxs, nsplit):
    import torch
    rng = np.random.default_rng(sum(ctxs) + nsplit)
    T = len(ctxs)
    max_pos = max(ctxs) + 16
    max_blocks = (max_pos + 15) // 16 + 1
    nblk = sum((c + 15) // 16 for c in ctxs) + 4
    perm = rng.permutation(nblk)  # physical blocks scattered over the pool
    bt = np.zeros((T, max_blocks), dtype=np.int32)
    used = 0
    for t, c in enumerate(ctxs):
        nb = (c + 15) // 16
        bt[t, :nb] = perm[used:used + nb]
        used += nb
    kc = (rng.standard_normal((nblk, HK, 16, D)) * 0.5).astype(np.float16)
    vc = rng.standard_normal((nblk, HK, 16, D)).astype(np.float16)
    qkv = rng.standard_normal((T, (HQ + 2 * HK) * D)).astype(np.float32)
    pos = np.array([c - 1 for c in ctxs], dtype=np.int32)  # newest position of each sequence
    slot = np.array([bt[t, p // 16] * 16 + p % 16 for t, p in enumerate(pos)], dtype=np.int32)
    seq_of = np.arange(T, dtype=np.int32)
    table = _rope_table(max_pos, D)
    # reference (before the kernel appends the new k / v)
    ref = np.zeros((T, HQ, D))
    for t in range(T):
        p = int(pos[t])
        q = _f16(_rope(qkv[t, :HQ * D].reshape(HQ, D).astype(np.float64), table[p]))
        kn = _f16(_rope(qkv[t, HQ * D:(HQ + HK) * D].reshape(HK, D).astype(np.float64), table[p]))
        vn = _f16(qkv[t, (HQ + HK) * D:].reshape(HK, D).astype(np.float64))
        kk = kc[bt[t, :(p // 16) + 1]].transpose(1, 0, 2, 3).reshape(HK, -1, D)[:, :p + 1].astype(np.float64)
        vv = vc[bt[t, :(p // 16) + 1]].transpose(1, 0, 2, 3).reshape(HK, -1, D)[:, :p + 1].astype(np.float64)
        kk[:, p] = kn
        vv[:, p] = vn
        for h in range(HQ):
            g = h // (HQ // HK)
            s = kk[g] @ q[h] / np.sqrt(D)
            w = np.exp(s - s.max())
            ref[t, h] = (w / w.sum()) @ vv[g]
    dev = {name: torch.from_numpy(np.ascontiguousarray(a)).cuda()
           for name, a in dict(qkv=qkv, table=table, pos=pos, slot=slot, seq=seq_of, bt=bt,
                               kc=kc.view(np.int16), vc=vc.view(np.int16)).items()}
    o = torch.empty((T, HQ, D), dtype=torch.float32, device="cuda")
    check_engine(engine_lib().msw_attention_decode(
        dev["qkv"].data_ptr(), dev["table"].data_ptr(), T, dev["pos"].data_ptr(), dev["slot"].data_ptr(),
        dev["seq"].data_ptr(), dev["bt"].data_ptr(), max_blocks, dev["kc"].data_ptr(), dev["vc"].data_ptr(),
        HQ, HK, D, nsplit, o.data_ptr(), None))
    got = o.cpu().numpy()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 2e-3, f"attention error {err:.3g}"
    # the new k / v were appended at slot[t] (fp16)
    kc_after = dev["kc"].cpu().numpy().view(np.float16)
    for t in range(T):
        p = int(pos[t])
        kn = _rope(qkv[t, HQ * D:(HQ + HK) * D].reshape(HK, D).astype(np.float64), table[p])
        got_k = kc_after[bt[t, p // 16], :, p % 16, :].astype(np.float64)
        assert np.abs(got_k - kn).max() <= 2e-3 * np.abs(kn).max() + 1e-3
