"""OPT-6.7B verify and OPT-125M draft-step time with GEMM debug flags (sb_debug_gemm_pdl): python scripts/opt_ab_dbg.py F1 F2 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
flags = [int(a) for a in sys.argv[1:]] or [0, 4]
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["opt-6.7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["opt-125m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=16, max_k=8, prompt_len=128,
                 max_new=128)
lib = N.load()
for b, k in [(1, 8), (4, 7), (8, 3), (8, 7), (16, 4)]:
    row = []
    for f in flags:
        lib.sb_debug_gemm_pdl(0, 0, f)
        v = min(eng.time_verify(b, k, ctx=192, reps=20) for _ in range(3))
        d = min(eng.time_draft_step(b, ctx=192, reps=50) for _ in range(2)) * 1e3
        row.append(f"flags={f}: verify {v:.3f} ms, draft {d:.1f} us")
    lib.sb_debug_gemm_pdl(0, 0, 0)
    print(f"b={b} k={k} | " + " | ".join(row), flush=True)
