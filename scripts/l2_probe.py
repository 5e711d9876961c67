"""Is the 68M draft's weight stream L2-resident across draft steps?  Draft step time
(and its lm_head + selection part: every layer kernel skipped) with the weight TMA
loads forced evict-first (1) vs evict-last (2) via SB_GEMM_W_L2HINT (one process per
setting: the env is read once).  Equal times = the weights come from HBM either way."""
import os, subprocess, sys

if len(sys.argv) == 1:
    for h in ("1", "2"):
        subprocess.run([sys.executable, __file__, h], env={**os.environ, "SB_GEMM_W_L2HINT": h}, check=True)
    sys.exit(0)
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
for b in (1, 8):
    full = eng.time_draft_step(b, ctx=192, reps=200) * 1e3
    lib.sb_debug_skip(31)
    head = eng.time_draft_step(b, ctx=192, reps=200) * 1e3
    lib.sb_debug_skip(0)
    print(f"hint={sys.argv[1]} b={b}: draft step {full:.2f} us, lm_head+select only {head:.2f} us", flush=True)
