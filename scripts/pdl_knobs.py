"""A/B of the GEMM's PDL behaviour (sb_debug_gemm_pdl) on the 7B verify forward."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=16, max_k=8, prompt_len=128,
                 max_new=128)
lib = N.load()
for b, k in [(8, 3), (1, 8), (16, 8)]:
    row = []
    for pre, late in [(0, 0), (1, 0), (2, 0), (4, 0), (0, 1), (2, 1)]:
        lib.sb_debug_gemm_pdl(pre, late, 0)
        ts = [eng.time_verify(b, k, ctx=192, reps=20) for _ in range(2)]
        row.append(f"pre={pre},late={late}: {min(ts):.3f}")
    lib.sb_debug_gemm_pdl(0, 0, 0)
    print(f"b={b} k={k} | " + " | ".join(row), flush=True)
