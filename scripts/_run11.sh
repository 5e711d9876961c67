timeout 600 python scripts/ab_dbg.py 0 1024 > gpurun_out/ab_pf.txt 2>&1; cat gpurun_out/ab_pf.txt
SB_ATTN_L2PF=1 timeout 600 python scripts/ab_dbg.py 0 > gpurun_out/ab_l2pf.txt 2>&1; cat gpurun_out/ab_l2pf.txt
