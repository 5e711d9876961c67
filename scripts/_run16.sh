SB_LIB=ab/old.so timeout 300 python -m pytest tests/test_gpu_gqa_shapes.py -q -x -p no:cacheprovider 2>&1 | tail -1
SB_LIB=ab/new.so timeout 300 python -m pytest tests/test_gpu_gqa_shapes.py -q -x -p no:cacheprovider 2>&1 | tail -1
CUDA_LAUNCH_BLOCKING=1 SB_DEBUG=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -c "
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.presets import example_trace
dev=torch.device('cuda:0')
tgt = Decoder(CONFIGS['llama-2-7b'], dtype='bf16', device=dev, init='device', max_pos=320)
drf = Decoder(CONFIGS['llama-68m'], dtype='bf16', device=dev, seed=1, init='device', max_pos=320)
eng = SpecEngine(tgt, drf, mode='injected', acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128, max_new=128, autotune=False)
from paper_2310_18813_b200.engine import SequenceState
st=[SequenceState(request_id=i, target_len=16) for i in range(8)]
eng.generate(st, 3); torch.cuda.synchronize(); print('ok')
" 2>&1 | grep -v "^=========     at\|^=========  *$" | head -40
