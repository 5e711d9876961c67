"""Draft step and whole-iteration time (graph replay) with the small-token GEMM on / off:
python scripts/small_gemm_ab.py {0|1}  (sb_set_small_gemm, set before any capture)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
on = int(sys.argv[1])
lib = N.load()
lib.sb_set_small_gemm(on)
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=32, max_k=8, prompt_len=128,
                 max_new=128)
ds = {b: min(eng.time_draft_step(b, ctx=192, reps=20) for _ in range(3)) * 1e3 for b in (1, 2, 4, 8, 16, 32)}
print(f"small_gemm={on} draft step us: " + " ".join(f"b={b}:{v:.1f}" for b, v in ds.items()), flush=True)
row = []
for b, k in [(1, 8), (4, 7), (8, 3), (8, 7), (16, 4)]:
    _stage_context(eng, b, k, 192)
    g = eng._graph(b, k)
    with torch.cuda.stream(eng.stream):
        for _ in range(3):
            _stage_context(eng, b, k, 192)
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            _stage_context(eng, b, k, 192)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
    row.append(f"b={b},k={k}: {min(ts):.3f}")
print(f"small_gemm={on} iteration ms: " + " | ".join(row), flush=True)
