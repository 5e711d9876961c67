import sys; sys.path.insert(0, '.')
import numpy as np, torch
from oracle import model_ref
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
N.load(); N.init_device()
dev = torch.device('cuda:0')
tgt = Decoder(CONFIGS["tiny-target"], dtype="bf16", device=dev, seed=1, init="host", max_pos=512)
ref = model_ref.LlamaRef(tgt.masters, 8, 8, 1e-5, max_pos=512, dtype=torch.float64, bf16_emulation=True)
ref32 = model_ref.LlamaRef(tgt.masters, 8, 8, 1e-5, max_pos=512, dtype=torch.float64, bf16_emulation=False)
b, P = 3, 21
ids = np.random.default_rng(0).integers(0, 32000, size=(b, P)).astype(np.int32)
for backend in (1, 2):
    N.call("sb_set_gemm_backend", backend)
    kv = tgt.new_kv(4, 256)
    T = b * P
    ws = torch.zeros(tgt.workspace_bytes(T), device=dev, dtype=torch.uint8)
    logits = torch.zeros(T, 32000, device=dev)
    slots = torch.arange(4, dtype=torch.int32, device=dev)
    pos = torch.arange(P, dtype=torch.int32, device=dev).repeat(b)
    tgt.forward(kv, torch.as_tensor(ids.reshape(-1), device=dev), slots, pos, b, P, logits, N.LOGITS_ALL, ws)
    torch.cuda.synchronize()
    g = logits.cpu().numpy().reshape(b, P, -1)
    w = ref.forward(list(ids[0]), list(range(P)), ref.new_cache())
    w32 = ref32.forward(list(ids[0]), list(range(P)), ref32.new_cache())
    print("backend", backend, "gpu absmax", np.abs(g[0]).max(), "ref absmax", np.abs(w).max(), np.abs(w32).max(),
          "rel", np.abs(g[0]-w).max()/np.abs(w).max(), "rel32", np.abs(g[0]-w32).max()/np.abs(w32).max(), "nan", np.isnan(g).sum())
