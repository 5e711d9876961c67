"""Verify timing with and without the measured GEMM autotuning (7B + 68M)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
lib = N.load()
grid = [(1, 3), (1, 8), (8, 1), (8, 3), (8, 8), (16, 3), (16, 8), (32, 3)]
for tuned in (0, 1):
    lib.sb_gemm_autotune_clear()
    t0 = time.perf_counter()
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=32, max_k=8, prompt_len=128,
                     max_new=128, autotune=bool(tuned))
    t_init = time.perf_counter() - t0
    r = [f"b{b}k{k}={eng.time_verify(b, k, ctx=192, reps=10):.3f}" for b, k in grid]
    d = [f"b{b}={eng.time_draft_step(b, ctx=192, reps=30) * 1e3:.1f}us" for b in (1, 8)]
    print(f"autotune={tuned} (engine init {t_init:.1f}s): verify ms " + " ".join(r) + " | draft " + " ".join(d), flush=True)
    if tuned:
        tt = eng.tuning["target"]
        print("tuned:", {f"{n}@{T}": v[:2] for (n, T), v in sorted(tt.items()) if T in (4, 32, 72, 144)}, flush=True)
