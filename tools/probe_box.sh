#!/bin/bash
# One-shot probe of the GPU box: devices, host cores, memory, NCCL, numpy speed.
mkdir -p gpurun_out
{
nvidia-smi -L
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Socket|MHz' ; free -g | head -2
python -c "import torch; print('devs', torch.cuda.device_count()); p=torch.cuda.get_device_properties(0); print(p.name, p.multi_processor_count, p.total_memory, getattr(p,'L2_cache_size',None))"
python -c "import torch; print('nccl', torch.cuda.nccl.version())"
python - <<'PY'
import time, numpy as np
t=time.time(); r=np.random.default_rng(np.random.SeedSequence(0, spawn_key=(2,0,0))); x=r.standard_t(3, 1<<20); print('t3 1M', time.time()-t)
PY
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
