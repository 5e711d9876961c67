"""gate/up (silu), qkv (store) and down (residual add) GEMM epilogues: 4-byte row emit (dbg 0) vs wide 16-byte emit (dbg 4) vs staging only
(dbg 2): per-CTA trace medians (us) and bit-identity of the outputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2310_18813_b200 import _native as N
dev = torch.device("cuda:0")
lib = N.load()
lib.sb_init()
buf = torch.zeros(8 + 8 * 100000, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream
for Nw, K, EPI, cols in ((22016, 4096, N.EPI_SILU_MUL, 11008), (12288, 4096, N.EPI_STORE, 12288),
                        (4096, 11008, N.EPI_RESID_ADD, 4096)):
  w = (torch.randn(Nw, K, device=dev) * 0.02).to(torch.bfloat16)
  for M in (9, 16, 32, 64, 128, 192, 288, 1016):
      x = torch.randn(M, K, device=dev).to(torch.bfloat16)
      outs = {}
      for dbg in (0, 4, 2):
          y = torch.zeros(M, cols, device=dev, dtype=torch.float32 if EPI == N.EPI_RESID_ADD else torch.bfloat16)
          lib.sb_debug_gemm_pdl(0, 0, dbg)
          for _ in range(3):
              N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, EPI, N.GEMM_TC, None, 0, st)
          torch.cuda.synchronize()
          outs[dbg] = y.clone()
          e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
          e0.record()
          for _ in range(20):
              N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, EPI, N.GEMM_TC, None, 0, st)
          e1.record(); e1.synchronize()
          buf.zero_()
          lib.sb_debug_cta_trace(N.ptr(buf))
          N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, EPI, N.GEMM_TC, None, 0, st)
          lib.sb_debug_cta_trace(None)
          torch.cuda.synchronize()
          n = int(buf[0].item())
          raw = buf[8:8 + 8 * n].view(n, 8).cpu().numpy().astype(np.int64)
          t0 = raw[:, 2].min()
          t = (raw[:, 2:7] - t0) / 1e3
          epi_d = t[:, 4] - t[:, 3]
          print(f"epi={EPI} M={M:5d} dbg={dbg}: ctas {n} epi med {np.median(epi_d):6.2f} p90 {np.percentile(epi_d, 90):6.2f} "
                f"total {t[:, 4].max():7.2f} | mean launch {e0.elapsed_time(e1) / 20 * 1e3:7.2f} us", flush=True)
      print(f"epi={EPI} M={M:5d} wide == row emit: {bool(torch.equal(outs[0], outs[4]))}", flush=True)
lib.sb_debug_gemm_pdl(0, 0, 0)
