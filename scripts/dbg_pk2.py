"""Debug: persistent forward intermediates vs torch on a 1-layer decoder."""
import sys, os; sys.path.insert(0, '.')
from dataclasses import replace
import torch, numpy as np
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
dev = torch.device('cuda:0')
name = os.environ.get("CFG", "tiny-target")
L = int(os.environ.get("L", "1"))
cfg = replace(CONFIGS[name], n_layers=L)
dec = Decoder(cfg, dtype="bf16", device=dev, init="device", max_pos=512)
b, q = int(os.environ.get("B", "2")), int(os.environ.get("Q", "3"))
T = b * q
H, nq, nkv, hd, ffn, V = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn, cfg.vocab
qd, qkv_n = nq * hd, (nq + 2 * nkv) * hd
ws = torch.zeros(dec.workspace_bytes(T), device=dev, dtype=torch.uint8)
def al(x): return (x + 255) // 256 * 256
tn = max(16, (T + 15) // 16 * 16)
offs = {}
o = 0
for nm, sz in [("sync", 4 * 1026), ("scratch", 148 * tn * 128 * 4), ("resid", T * H * 4), ("xn", T * H * 2),
               ("qkv", T * qkv_n * 2), ("qr", T * qd * 2), ("attn", T * qd * 2), ("act", T * ffn * 2),
               ("last", T * H * 2), ("amv", ((V + 127) // 128) * T * 4), ("ami", ((V + 127) // 128) * T * 4),
               ("xb", T * H * 2), ("npart", ((H + 127) // 128) * 8 * T * 4)]:
    offs[nm] = (o, sz); o += al(sz)
def buf(nm, dt, shape):
    a, sz = offs[nm]
    return ws[a:a + sz].view(dt).view(*shape)
ids = torch.randint(0, V, (T,), dtype=torch.int32, device=dev)
pos = torch.arange(q, dtype=torch.int32, device=dev).repeat(b)
slots = torch.arange(b, dtype=torch.int32, device=dev)
kv = dec.new_kv(b, 64)
lg = torch.zeros(T, V, device=dev)
mode = N.LOGITS_ALL if os.environ.get("LM", "1") == "1" else N.LOGITS_NONE
dec.forward(kv, ids, slots, pos, b, q, lg if mode == N.LOGITS_ALL else None, mode, ws)
torch.cuda.synchronize()
print("sync words", ws[:16].view(torch.int32).tolist())
# ---- torch reference
f = lambda t: t.float()
bf = lambda t: t.to(torch.bfloat16).float()
x = f(dec.embed[ids.long()])
def rel(a, b_):
    return ((a - b_).abs().max() / max(b_.abs().max().item(), 1e-9)).item()
cos, sin = dec.rope_cos, dec.rope_sin
for l in range(L):
    lay = dec.layers[l]
    inv = torch.rsqrt((x * x).mean(1, keepdim=True) + cfg.rms_eps)
    qkv = bf(bf(x) @ f(lay["w_qkv"]).T * inv)
    qq = qkv[:, :qd].view(T, nq, hd); kk = qkv[:, qd:qd + nkv * hd].view(T, nkv, hd); vv = qkv[:, qd + nkv * hd:].view(T, nkv, hd)
    c = cos[pos.long()][:, None, :]; s = sin[pos.long()][:, None, :]
    def rot(t):
        h = hd // 2
        x0, x1 = t[..., :h], t[..., h:]
        return bf(torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], -1))
    qr, kr = rot(qq), rot(kk)
    if l == L - 1 and mode == N.LOGITS_NONE:
        print("qr rel", rel(f(buf("qr", torch.bfloat16, (T, qd))), qr.view(T, qd)))
    kc = f(kv.k[l]); vc = f(kv.v[l])
    for t in range(T):
        sl, p_ = t // q, pos[t].item()
        if l == L - 1: pass
    print(f"L{l} K cache rel", rel(torch.stack([kc[t // q, :, pos[t]] for t in range(T)]), kr),
          "V cache rel", rel(torch.stack([vc[t // q, :, pos[t]] for t in range(T)]), vv))
    att = torch.zeros(T, nq, hd, device=dev)
    grp = nq // nkv
    for t in range(T):
        sq, p_ = t // q, pos[t].item()
        for h in range(nq):
            K = kc[sq, h // grp, :p_ + 1]; Vv = vc[sq, h // grp, :p_ + 1]
            w = torch.softmax(qr[t, h] @ K.T / hd ** 0.5, 0)
            att[t, h] = w @ Vv
    att = bf(att.view(T, qd))
    if l == L - 1 and mode == N.LOGITS_NONE:
        print("attn rel", rel(f(buf("attn", torch.bfloat16, (T, qd))), att))
    x = x + att @ f(lay["w_o"]).T
    inv = torch.rsqrt((x * x).mean(1, keepdim=True) + cfg.rms_eps)
    gu = bf(x) @ f(lay["w_gu"]).T * inv
    g, u = gu[:, 0::2], gu[:, 1::2]
    act = bf(g / (1 + torch.exp(-g)) * u)
    if l == L - 1 and mode == N.LOGITS_NONE:
        print("act rel", rel(f(buf("act", torch.bfloat16, (T, ffn))), act))
    x = x + act @ f(lay["w_down"]).T
if mode == N.LOGITS_NONE:
    print("resid rel", rel(buf("resid", torch.float32, (T, H)), x))
    print("xb rel", rel(f(buf("xb", torch.bfloat16, (T, H))), bf(x)))
    ss = (x * x).sum(1)
    npt = buf("npart", torch.float32, (-1,))[: ((H + 127) // 128) * T].view(-1, T).sum(0)
    print("norm partial rel", rel(npt, ss) if L > 0 else rel(buf("npart", torch.float32, (-1,))[:T], ss))
else:
    inv = torch.rsqrt((x * x).mean(1, keepdim=True) + cfg.rms_eps)
    ref = bf(x) @ f(dec.lm_head).T * inv
    print("logits rel", rel(lg, ref))
