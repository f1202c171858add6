timeout 120 ncu --metrics gpu__time_duration.sum -c 1 python -c "
import os
print({k: v[:80] for k, v in os.environ.items() if any(t in k for t in ('INJ', 'NSIGHT', 'NV_', 'PRELOAD', 'CUDA', 'TOOL', 'NCU'))})
import torch; torch.zeros(1, device='cuda'); print('done')
" 2>&1 | grep -v "^==PROF==" | head -20
