"""Verify-forward roofline crossover (north_star: HBM-bound at small b(k+1),
tensor-bound at large): time one target verify (CUDA graph replay) over a
(b, k) grid and report achieved GB/s (algorithmic bytes) and
TFLOP/s (2 * params * T + attention) against MEASURED_PEAKS.json."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm, tf = peaks["hbm_gbs"], peaks["bf16_tflops"]
name = os.environ.get("CFG", "llama-2-7b")
dev = torch.device("cuda:0")
cfg = CONFIGS[name]
tgt = Decoder(cfg, dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=64, max_k=8, prompt_len=128,
                 max_new=128)
ctx = 192
if os.environ.get("SB_PERSISTENT") == "1":
    from paper_2310_18813_b200 import _native as N
    N.load().sb_set_persistent(1)
W = cfg.streamed_bytes_per_forward(2)
params = W / 2
rows = []
grid_b = [int(x) for x in os.environ.get("XB", "1,2,4,8,16,32,64").split(",")]
grid_k = [int(x) for x in os.environ.get("XK", "1,3,8").split(",")]
for b in grid_b:
    for k in grid_k:
        T = b * (k + 1)
        ms = eng.time_verify(b, k, ctx=ctx, reps=10)
        byts = W + cfg.kv_bytes_per_token(2) * (b * ctx + T) + 4 * cfg.vocab * T + 2 * cfg.hidden * T
        flops = 2 * params * T + 4 * cfg.n_layers * cfg.hidden * (k + 1) * b * (ctx + (k + 2) / 2)
        r = {"b": b, "k": k, "T": T, "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1),
             "TFLOPs": round(flops / ms / 1e9, 1), "intensity_flop_per_byte": round(flops / byts, 1),
             "frac_hbm": round(byts / ms / 1e6 / hbm, 3), "frac_tensor": round(flops / ms / 1e9 / tf, 3)}
        rows.append(r)
        print(json.dumps(r), flush=True)
out = {"target": name, "ctx": ctx, "peak_hbm_gbs": hbm, "peak_bf16_tflops": tf,
       "ridge_flop_per_byte": round(tf * 1e12 / (hbm * 1e9), 1), "rows": rows}
print("SUMMARY " + json.dumps(out))
