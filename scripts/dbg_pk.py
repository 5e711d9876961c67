import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
dev=torch.device('cuda:0')
for name in ["tiny-target","llama-68m"]:
    cfg=CONFIGS[name]
    dec=Decoder(cfg,dtype="bf16",device=dev,init="device",max_pos=512)
    for b,q in [(1,1),(2,3),(3,9),(8,4),(8,12),(4,16)]:
        kv=dec.new_kv(b,128); T=b*q
        ws=torch.zeros(dec.workspace_bytes(T),device=dev,dtype=torch.uint8)
        ids=torch.randint(0,32000,(T,),dtype=torch.int32,device=dev)
        pos=torch.arange(q,dtype=torch.int32,device=dev).repeat(b)
        slots=torch.arange(b,dtype=torch.int32,device=dev)
        lg=torch.zeros(T,32000,device=dev)
        try:
            dec.forward(kv,ids,slots,pos,b,q,lg,N.LOGITS_ALL,ws); torch.cuda.synchronize(); print(name,b,q,"ok",flush=True)
        except Exception as e: print(name,b,q,"ERR",e,flush=True)
