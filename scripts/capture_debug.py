"""Find the native call after which a CUDA graph capture is invalidated: run
the test_gpu_model sequence that fails and check cudaStreamIsCapturing after
every native call."""
import ctypes, glob, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_model as T

cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*")
rt = ctypes.CDLL(cands[0])
def cap_status(st):
    s = ctypes.c_int(-1)
    rc = rt.cudaStreamIsCapturing(ctypes.c_void_p(st), ctypes.byref(s))
    return rc, s.value
orig = N.call
state = {"bad": False}
def call(name, *args):
    st = args[-1] if args and isinstance(args[-1], int) else None
    before = cap_status(st) if st else None
    try:
        return orig(name, *args)
    finally:
        if st:
            after = cap_status(st)
            if before and before[1] == 1 and after[1] != 1 and not state["bad"]:
                state["bad"] = True
                print(f"CAPTURE INVALIDATED by {name}: before={before} after={after}", flush=True)
            elif before and before[1] == 2 and not state["bad"]:
                state["bad"] = True
                print(f"capture already invalid before {name}", flush=True)
N.call = call
dev = torch.device("cuda:0")
seq = [(T.test_host_init_reproduced_by_oracle, {}), (T.test_forward_logits_match_oracle, {"dtype": "fp32"}),
       (T.test_forward_logits_match_oracle, {"dtype": "bf16"})] + \
      [(T.test_fp32_greedy_spec_equals_cpu_greedy, {"k": k}) for k in (0, 1, 3, 8)] + \
      [(T.test_fp32_spec_is_batch_invariant_and_graph_consistent, {})]
for fn, kw in seq:
    try:
        fn(dev, **kw)
        print("ok", fn.__name__, kw, flush=True)
    except Exception as e:
        print("FAIL", fn.__name__, kw, type(e).__name__, str(e)[:200], flush=True)
        break
