"""One config of K1 for ncu: warm replays, then a few profiled launches (b, k from argv)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
sys.argv.append("--no-run")
import draft_loop_time as T  # noqa: E402
from paper_2310_18813_b200 import _native as N  # noqa: E402

b, k = int(sys.argv[1]), int(sys.argv[2])
d1_ids, d1_pos, d_base = T.setup(b)
v_ids = torch.zeros(b * (k + 1), **T.i32)
ds_ids = torch.zeros(b, **T.i32)
ds_pos = torch.zeros(b, **T.i32)
for _ in range(6):
    rc = T.lib.sb_draft_loop(C.byref(T.drf.struct), C.byref(T.kv.struct), N.ptr(T.packed), b, k, N.ptr(d1_ids),
                             N.ptr(d1_pos), N.ptr(T.slots), N.ptr(d_base), N.ptr(v_ids), N.ptr(ds_ids), N.ptr(ds_pos),
                             N.ptr(T.ws), T.ws.numel(), N.ptr(T.sync), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
torch.cuda.synchronize()
print("ok")
