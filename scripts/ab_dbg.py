"""A/B of GEMM debug flags (sb_debug_gemm_pdl flags) on the 7B verify forward: python scripts/ab_dbg.py F1 F2 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
flags = [int(a) for a in sys.argv[1:]] or [0, 8]
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
cells = [tuple(int(x) for x in c.split(",")) for c in os.environ.get("CELLS", "").split()] or \
    [(1, 8), (2, 7), (4, 7), (8, 3), (16, 8), (32, 8)]
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=max(32, max(b for b, _ in cells)),
                 max_k=8, prompt_len=128, max_new=128)
lib = N.load()
if os.environ.get("ATTN_SPLITS"):
    lib.sb_set_attention_splits(int(os.environ["ATTN_SPLITS"]))
for b, k in cells:
    row = []
    for f in flags:
        lib.sb_debug_gemm_pdl(0, 0, f)
        ts = [eng.time_verify(b, k, ctx=192, reps=20) for _ in range(3)]
        row.append(f"flags={f}: {min(ts):.3f}")
    lib.sb_debug_gemm_pdl(0, 0, 0)
    d = [eng.time_draft_step(b, ctx=192, reps=20) for _ in range(2)]
    print(f"b={b} k={k} | " + " | ".join(row) + f" | draft step {min(d)*1e3:.1f} us", flush=True)
