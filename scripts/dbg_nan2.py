import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from dataclasses import replace
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
dev = torch.device("cuda:0")
tgt = Decoder(replace(CONFIGS["llama-2-7b"], n_layers=2), dtype="bf16", device=dev, seed=3, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=4, init="device", max_pos=320)
b, k = 8, 2
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=64,
                 max_new=32, seed=7, use_graphs=False, autotune=False)
_stage_context(eng, b, k, 150)
kv_ref = drf.new_kv(eng.max_batch, eng.ctx_max)
kv_ref.k.copy_(eng.kv_d.k); kv_ref.v.copy_(eng.kv_d.v)
logits = torch.zeros(b, drf.cfg.vocab, device=dev)
drf.forward(kv_ref, eng.d1_ids, eng.slots, eng.d1_pos, b, 2, logits, N.LOGITS_LAST, eng.workspace)
torch.cuda.synchronize()
print("before: nan rows", torch.isnan(logits).any(1).nonzero().flatten().tolist(), flush=True)
snap = logits.clone()
rc = N.load().sb_draft_loop(C.byref(drf.struct), C.byref(eng.kv_d.struct), b, k, N.ptr(eng.d1_ids), N.ptr(eng.d1_pos),
                            N.ptr(eng.slots), N.ptr(eng.d_base), N.ptr(eng.v_ids), N.ptr(eng.ds_ids), N.ptr(eng.ds_pos),
                            N.ptr(eng.workspace), eng.workspace.numel(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("rc", rc, "after: nan rows", torch.isnan(logits).any(1).nonzero().flatten().tolist(),
      "changed", (logits != snap).any().item(), flush=True)
print("ws", eng.workspace.data_ptr(), eng.workspace.numel(), "logits", logits.data_ptr(), "kv_ref", kv_ref.k.data_ptr())
print("v_ids", eng.v_ids[: b * (k + 1)].view(b, k + 1).tolist())
