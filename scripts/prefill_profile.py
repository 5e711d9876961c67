"""Per-stage time of the 7B prefill forward (b=8 prompts of 127 tokens, T=1016):
eager launches with an event after every kernel (sb_profile_forward)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
lib = N.load(); N.init_device()
b, q = int(os.environ.get("B", "8")), 127
T = b * q
kv = tgt.new_kv(b, 272)
ws = torch.zeros(tgt.workspace_bytes(T), device=dev, dtype=torch.uint8)
ids = torch.randint(0, 32000, (T,), dtype=torch.int32, device=dev)
pos = torch.arange(q, dtype=torch.int32, device=dev).repeat(b)
slots = torch.arange(b, dtype=torch.int32, device=dev)
if os.environ.get("TUNE") == "1":
    print("tuned:", {k: v for k, v in tgt.autotune([T]).items()})
buf = C.create_string_buffer(8192)
for rep in range(3):
    rc = lib.sb_profile_forward(C.byref(tgt.struct), C.byref(kv.struct), ids.data_ptr(), slots.data_ptr(), pos.data_ptr(),
                                b, q, None, N.LOGITS_NONE, ws.data_ptr(), ws.numel(),
                                torch.cuda.current_stream().cuda_stream, buf, 8192)
parts = [p.split("=") for p in buf.value.decode().strip(";").split(";")]
tot = sum(float(v) for _, v in parts)
print(f"prefill T={T}: eager-with-events total {tot:.2f} ms: " + " ".join(f"{t}={float(v):.2f}" for t, v in parts))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        tgt.forward(kv, ids, slots, pos, b, q, None, N.LOGITS_NONE, ws)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); g.replay(); g.replay(); e1.record(); e1.synchronize()
print(f"graph replay: {e0.elapsed_time(e1) / 3:.2f} ms per prefill forward")
