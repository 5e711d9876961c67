"""One eager 7B verify forward between cudaProfilerStart/Stop (for ncu --profile-from-start off):
python scripts/ncu_verify.py [b k]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
b, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 3)
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=max(b, 8), max_k=8, prompt_len=128,
                 max_new=128)
_stage_context(eng, b, k, 192)
fn = lambda: eng.target.forward(eng.kv_t, eng.v_ids, eng.slots, eng.v_pos, b, k + 1, eng.t_logits, N.LOGITS_ALL,
                                eng.workspace)
fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
