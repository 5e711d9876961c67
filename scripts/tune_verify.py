"""Verify-forward time (CUDA graph replay) under tcgen05 GEMM tuning overrides
(sb_gemm_tune: CTAs per SM, max stages, K splits; 0 = automatic)."""
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
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128,
                 max_new=128)
lib = N.load()
cfgs = [tuple(int(v) for v in c.split(":")) for c in os.environ.get(
    "TV", "0:0:0,1:0:0,2:3:0,2:4:0,2:5:0,2:6:0,1:6:0,1:8:0,2:4:4,2:4:2,1:0:4").split(",")]
for c in cfgs:
    lib.sb_gemm_tune(*c)
    r = [f"b{b}k{k}={eng.time_verify(b, k, ctx=192, reps=20):.3f}" for b, k in [(1, 3), (8, 1), (8, 3), (8, 8)]]
    print(f"tune={c}: verify ms " + " ".join(r), flush=True)
lib.sb_gemm_tune(0, 0, 0)
