"""One standalone tcgen05 GEMM launch for ncu (after warm-up): python scripts/ncu_gemm1.py M N K epi"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
M, Nw, K, epi = (int(a) for a in sys.argv[1:5])
dev = torch.device("cuda:0")
lib = N.load(); lib.sb_init()
w = (torch.randn(Nw, K, device=dev) * 0.02).to(torch.bfloat16)
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
y = torch.zeros(M, Nw, device=dev)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
