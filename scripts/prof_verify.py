"""Profile target: eager verify forwards (7B, bf16) + draft steps for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context

b = int(os.environ.get("PB", "8")); k = int(os.environ.get("PK", "3"))
layers = int(os.environ.get("PL", "32"))
dev = torch.device("cuda:0")
cfg = CONFIGS["llama-2-7b"]
from dataclasses import replace
tgt = Decoder(replace(cfg, n_layers=layers), dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=max(8, b), max_k=max(8, k), prompt_len=128, max_new=128)
_stage_context(eng, b, k, 192)
for i in range(int(os.environ.get("PREPS", "3"))):
    tgt.forward(eng.kv_t, eng.v_ids, eng.slots, eng.v_pos, b, k + 1, eng.t_logits, N.LOGITS_ALL, eng.workspace)
    drf.forward(eng.kv_d, eng.ds_ids, eng.slots, eng.ds_pos, b, 1, eng.d_logits, N.LOGITS_LAST, eng.workspace)
torch.cuda.synchronize()
print("verify ms (graph):", eng.time_verify(b, k, ctx=192, reps=10), "draft step ms:", eng.time_draft_step(b, ctx=192, reps=10))
