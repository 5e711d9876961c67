"""Per-phase timeline of the persistent forward (globaltimer stamps per CTA)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import numpy as np, torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
dev = torch.device("cuda:0")
name = os.environ.get("CFG", "llama-2-7b"); L = int(os.environ.get("L", "4"))
b, k = int(os.environ.get("B", "8")), int(os.environ.get("K", "3"))
cfg = replace(CONFIGS[name], n_layers=L)
dec = Decoder(cfg, dtype="bf16", device=dev, init="device", max_pos=512)
q = k + 1; T = b * q; ctx = 192
kv = dec.new_kv(b, 256)
ws = torch.zeros(dec.workspace_bytes(T), device=dev, dtype=torch.uint8)
ids = torch.randint(0, cfg.vocab, (T,), dtype=torch.int32, device=dev)
pos = (torch.arange(q, dtype=torch.int32, device=dev) + ctx).repeat(b)
slots = torch.arange(b, dtype=torch.int32, device=dev)
lg = torch.zeros(T, cfg.vocab, device=dev)
G = torch.cuda.get_device_properties(0).multi_processor_count
nph = 1 + 5 * L + 1
tr = torch.zeros(G * nph * 8, dtype=torch.int64, device=dev)
lib = N.load()
for i in range(3):
    dec.forward(kv, ids, slots, pos, b, q, lg, N.LOGITS_ALL, ws)
lib.sb_debug_persistent_trace(tr.data_ptr())
dec.forward(kv, ids, slots, pos, b, q, lg, N.LOGITS_ALL, ws)
torch.cuda.synchronize()
lib.sb_debug_persistent_trace(None)
t = tr.view(G, nph, 8).cpu().numpy().astype(np.float64)
t0 = t[:, 0, 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
names = ["embed"] + [f"{n}{l}" for l in range(L) for n in ("qkv", "attn", "o", "gu", "down")] + ["lm"]
print(f"{name} L={L} b={b} k={k} T={T}: total {np.nanmax(t[:, -1, 3]):.1f} us")
for ph in range(nph):
    ws_ = t[:, ph, 1] - t[:, ph, 0]
    start = np.nanmin(t[:, ph, 1]); end = np.nanmax(t[:, ph, 3])
    first = t[:, ph, 2] - t[:, ph, 1]
    dur = t[:, ph, 3] - t[:, ph, 1]
    print(f"{names[ph]:>7}: span {start:8.1f}->{end:8.1f} ({end - start:6.1f} us)  barrier wait mean {np.nanmean(ws_):6.1f} "
          f"first-acc mean {np.nanmean(first) if np.isfinite(first).any() else 0:6.1f}  dur min/mean/max "
          f"{np.nanmin(dur):6.1f}/{np.nanmean(dur):6.1f}/{np.nanmax(dur):6.1f}")
# per-CTA detail for a few phases
kb = {"qkv": cfg.hidden // 64, "o": cfg.hidden // 64, "gu": cfg.hidden // 64, "down": cfg.ffn // 64}
nt = {"qkv": cfg.qkv_rows // 128, "o": cfg.hidden // 128, "gu": 2 * cfg.ffn // 128, "down": cfg.hidden // 128}
for ph, nm in [(1, "qkv"), (3, "o"), (5, "down")]:
    dur = t[:, ph, 3] - t[:, ph, 1]
    U = nt[nm] * kb[nm]
    ctas = min(G, (U + 3) // 4)
    order = np.argsort(-np.nan_to_num(dur))
    print(f"phase {names[ph]}: units {U} ctas {ctas}; slowest CTAs:")
    for c in order[:8]:
        s, e = c * U // ctas, (c + 1) * U // ctas
        segs = []
        u = s
        while u < e:
            tile = u // kb[nm]; a = u - tile * kb[nm]; se = min(e, (tile + 1) * kb[nm])
            segs.append(f"t{tile}[{a}:{se - tile * kb[nm]}]")
            u = se
        b0 = t[c, ph, 1]
        print(f"   cta {c:3d} dur {dur[c]:6.1f} first {t[c, ph, 2] - b0:6.1f} flagwait {t[c, ph, 4] - b0:6.1f}->{t[c, ph, 5] - b0:6.1f} "
              f"lastacc {t[c, ph, 6] - b0:6.1f} publish {t[c, ph, 7] - b0:6.1f} segs {' '.join(segs)}")
    print("   fastest:", " ".join(f"{c}:{dur[c]:.1f}" for c in order[-5:]))
